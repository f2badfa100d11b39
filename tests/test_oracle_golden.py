"""Pin the CPU oracle (oracle/radix.py) against the reference's golden vectors.

The vectors were produced by running the unmodified reference SessionTrie
(tests/golden/make_golden.py); every row/parent/matched/added/stats value and every
extracted trajectory must agree exactly before the oracle may judge the GPU.
"""

from oracle.radix import FlatOracle, RadixOracle


def test_radix_oracle_matches_reference_golden(trie_cases):
    assert len(trie_cases) > 300
    for case in trie_cases:
        o = RadixOracle()
        for ins, exp in zip(case["inserts"], case["results"]):
            got = o.insert(ins["tokens"], ins["origins"], ins["versions"], ins["completion_id"])
            assert (got.matched, got.row, got.parent, got.added) == (
                exp["matched"], exp["row"], exp["parent"], exp["added"]), case["name"]
            assert o.stats() == (exp["stored"], exp["naive"]), case["name"]
        ext = o.extract()
        assert [e[0] for e in ext] == [e["row"] for e in case["extract"]], case["name"]
        for (row, toks, mask, vers), e in zip(ext, case["extract"]):
            assert toks == e["tokens"]
            assert [int(m) for m in mask] == e["loss_mask"]
            assert vers == e["versions"]
        for row, p in case["paths"].items():
            toks, mask, vers = o.path(int(row))
            assert toks == p["tokens"] and [int(m) for m in mask] == p["loss_mask"] and vers == p["versions"]


def test_flat_oracle_matches_reference_golden(trie_cases):
    """flat rows + parent pointers reproduce the trie."""
    for case in trie_cases:
        f = FlatOracle()
        for ins, exp in zip(case["inserts"], case["results"]):
            got = f.insert(ins["tokens"], ins["origins"], ins["versions"])
            assert (got.matched, got.row, got.parent, got.added) == (
                exp["matched"], exp["row"], exp["parent"], exp["added"]), case["name"]
        assert (f.stored, f.naive) == (case["stored"], case["naive"])
        for row, p in case["paths"].items():
            mask, vers = f.meta[int(row)]
            assert list(f.seqs[int(row)]) == p["tokens"]
            assert [int(m) for m in mask] == p["loss_mask"] and vers == p["versions"]
