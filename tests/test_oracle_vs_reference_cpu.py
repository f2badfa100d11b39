"""The C restatement of the trie (oracle/radix_oracle.c, the checker every GPU parity test
uses) against the UNMODIFIED reference (rolloutlab.trie from baseline/_ref, installed by
tools/install_reference.sh) on seeded random record streams: branching off earlier
sequences at random depths, small vocabularies (long shared prefixes and collisions),
strict prefixes of stored sequences, exact re-records and metadata runs that change at
random positions.  Every insert's matched length / end node / added tokens, every
session's StorageStats, and extract() (order, tokens, loss masks, versions) must agree.
Complements the golden fixtures (tests/golden), which pin the same oracle to captured
outputs of the reference.  Skipped when baseline/_ref is absent."""

import numpy as np
import pytest

from oracle.cport import CRadixStore
from tools.refbench import reference_modules
from workloads import pack_records


def _stream(rng, n_sess, n_ins):
    sids, seqs, origins, versions = [], [], [], []
    ctx = {s: [] for s in range(n_sess)}
    for _ in range(n_ins):
        s = int(rng.integers(n_sess))
        prior = ctx[s]
        u = rng.random()
        vocab = 3 if rng.random() < 0.4 else 200
        if prior and u < 0.1:  # exact re-record
            seq = list(prior[int(rng.integers(len(prior)))])
        elif prior and u < 0.2:  # strict prefix of a stored sequence
            base = prior[int(rng.integers(len(prior)))]
            seq = base[: max(1, int(rng.integers(1, len(base) + 1)))]
        elif prior:  # branch off an earlier sequence at a random depth
            base = prior[int(rng.integers(len(prior)))]
            cut = int(rng.integers(0, len(base) + 1))
            seq = base[:cut] + rng.integers(0, vocab, int(rng.integers(1, 40))).tolist()
        else:
            seq = rng.integers(0, vocab, int(rng.integers(1, 60))).tolist()
        # runs: origin flips and version steps at random positions (versions non-decreasing)
        n = len(seq)
        org = np.zeros(n, np.int64)
        ver = np.zeros(n, np.int64)
        for _ in range(int(rng.integers(0, 4))):
            p = int(rng.integers(0, n))
            org[p:] ^= 1
        for _ in range(int(rng.integers(0, 3))):
            ver[int(rng.integers(0, n)):] += 1
        sids.append(s)
        seqs.append(seq)
        origins.append(org.tolist())
        versions.append(ver.tolist())
        ctx[s].append(seq)
    return sids, seqs, origins, versions


@pytest.mark.parametrize("seed", range(6))
def test_c_oracle_matches_unmodified_reference_random(seed):
    mods = reference_modules()
    if mods is None:
        pytest.skip("the unmodified reference is not installed in baseline/_ref (tools/install_reference.sh)")
    trie_mod, core = mods
    rng = np.random.default_rng(4200 + seed)
    n_sess = 10
    sids, seqs, origins, versions = _stream(rng, n_sess, 500)
    a, o = core.SpanOrigin.AGENT_INPUT, core.SpanOrigin.MODEL_OUTPUT
    tries = {s: trie_mod.SessionTrie(f"s{s}") for s in range(n_sess)}
    node_row = {s: {} for s in range(n_sess)}
    expect = []
    for k, s in enumerate(sids):
        res = tries[s].lpm_insert(seqs[k], [o if x else a for x in origins[k]], versions[k], completion_id=f"c{k}")
        rows = node_row[s]
        if res.node_id not in rows:
            rows[res.node_id] = len(rows)
        expect.append((res.matched_prefix_length, rows[res.node_id], res.added_tokens))

    st = CRadixStore()
    m, row, _par, add = st.insert_batch(*pack_records(sids, seqs, origins, versions), nthreads=2)
    for k in range(len(sids)):
        assert (int(m[k]), int(row[k]), int(add[k])) == expect[k], k

    for s in range(n_sess):
        ref_stats = tries[s].stats()
        stored, naive, nrows = st.stats(s)
        assert (stored, naive) == (ref_stats.stored_tokens, ref_stats.naive_tokens)
        assert nrows == len(node_row[s])
        ref_extract = tries[s].extract()  # every row ends an insert, so every row is marked
        assert st.lex_rows(s).tolist() == [node_row[s][nid] for nid, _ in ref_extract]
        for nid, traj in ref_extract:
            t, mk, v = st.export_row(s, node_row[s][nid])
            assert t.tolist() == list(traj.tokens)
            assert mk.tolist() == [int(x) for x in traj.loss_mask]
            assert v.tolist() == list(traj.version_tags)
