"""GPU parity: the B200 store against the reference golden vectors and the C oracle.

Everything here calls through the C ABI (libtmstore.so) on cuda:0.  Integer work, so
the bar is bit-exact: matched length, row (node id), chosen parent row, added tokens,
storage stats, export order and every token / loss-mask / version value.
"""

import numpy as np
import pytest

from oracle.cport import CRadixStore
from workloads import pack_records

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["default", "planner", "planner+roots"])
def store(request):
    """Every test runs on each walk schedule: the store default, the longest-first
    planner forced on, and the planner also resolving root rows."""
    import os

    from paper_2508_11553_b200 import DeviceStore

    env = {"default": {}, "planner": {"TM_PLAN_MIN": "1", "TM_PLAN_ROOTS": "0"},
           "planner+roots": {"TM_PLAN_MIN": "1", "TM_PLAN_ROOTS": "1"}}[request.param]
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = DeviceStore(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    yield s
    s.close()


def _origins(codes):
    from paper_2508_11553_b200 import SpanOrigin

    return [SpanOrigin.MODEL_OUTPUT if c else SpanOrigin.AGENT_INPUT for c in codes]


def test_golden_cases_through_session_trie(store, trie_cases):
    """Every golden stream through the drop-in SessionTrie, insert by insert."""
    from paper_2508_11553_b200 import SessionTrie, trajectory_to_line

    for case in trie_cases:
        trie = SessionTrie(case["session_id"], store=store)
        for ins, exp in zip(case["inserts"], case["results"]):
            r = trie.lpm_insert(ins["tokens"], _origins(ins["origins"]), ins["versions"], ins["completion_id"])
            assert (r.matched_prefix_length, r.node_id, r.added_tokens) == (exp["matched"], exp["row"], exp["added"]), case["name"]
            st = trie.stats()
            assert (st.stored_tokens, st.naive_tokens) == (exp["stored"], exp["naive"]), case["name"]
        assert trie.stats().dedup_ratio == case["dedup_ratio"]
        ext = trie.extract()
        assert [k for k, _ in ext] == [e["row"] for e in case["extract"]], case["name"]
        for (_, t), e in zip(ext, case["extract"]):
            assert trajectory_to_line(t) == e["line"]
        for row, p in case["paths"].items():
            t = trie.path_trajectory(int(row))
            assert t.tokens == p["tokens"]
            assert [int(m) for m in t.loss_mask] == p["loss_mask"] and t.version_tags == p["versions"]
        assert trie.check_well_formed() == []
        marked = trie.marked_nodes()
        assert [n.node_id for n in marked] == [e["row"] for e in case["extract"]]
        assert all(n.is_marked for n in marked)


def test_golden_cases_as_one_batch(store, trie_cases):
    """All golden streams in ONE record batch (sequential semantics across waves),
    including the parent rows the reference does not report."""
    sids, seqs, origins, versions = [], [], [], []
    base = [store.new_session() for _ in trie_cases]
    for s, case in zip(base, trie_cases):
        for ins in case["inserts"]:
            sids.append(s)
            seqs.append(ins["tokens"])
            origins.append(ins["origins"])
            versions.append(ins["versions"])
    sid_a, tok, off, roff, rs, ro, rv = pack_records(sids, seqs, origins, versions)
    res = store.record_packed(sid_a, tok, off[:-1], np.diff(off), roff, rs, ro, rv)
    k = 0
    for s, case in zip(base, trie_cases):
        for exp in case["results"]:
            assert (res.matched[k], res.local[k], res.parent_local[k], res.added[k]) == (
                exp["matched"], exp["row"], exp["parent"], exp["added"]), case["name"]
            k += 1
        stored, naive, _ = store.session_stats(s)
        assert (stored, naive) == (case["stored"], case["naive"])


def _random_sessions(rng, n_sess, n_ins, vocab, max_new):
    sids, seqs, origins, versions = [], [], [], []
    ctx = {s: [[]] for s in range(n_sess)}
    for _ in range(n_ins):
        s = int(rng.integers(n_sess))
        base = ctx[s][int(rng.integers(len(ctx[s])))]
        r = rng.random()
        if r < 0.1 and len(base) > 1:
            seq = base[: int(rng.integers(1, len(base)))]          # strict prefix
        elif r < 0.2 and len(base) > 0:
            seq = list(base)                                        # duplicate
        elif r < 0.35 and len(base) > 2:                            # branch inside
            cut = int(rng.integers(1, len(base)))
            seq = base[:cut] + rng.integers(0, vocab, int(rng.integers(1, max_new))).tolist()
        else:
            seq = base + rng.integers(0, vocab, int(rng.integers(1, max_new))).tolist()
        org = (rng.random(len(seq)) < 0.5).astype(int).tolist()
        ver = np.sort(rng.integers(0, 3, len(seq))).tolist()
        sids.append(s)
        seqs.append(seq)
        origins.append(org)
        versions.append(ver)
        ctx[s].append(seq)
    return sids, seqs, origins, versions


@pytest.mark.parametrize("vocab,max_new,n_sess,n_ins", [(4, 12, 30, 600), (151936, 700, 50, 800), (3, 200, 5, 300)])
def test_random_batches_vs_c_oracle(store, vocab, max_new, n_sess, n_ins):
    rng = np.random.default_rng(vocab * 7 + n_ins)
    sids, seqs, origins, versions = _random_sessions(rng, n_sess, n_ins, vocab, max_new)
    ora = CRadixStore()
    rec = pack_records(sids, seqs, origins, versions)
    om, orow, opar, oadd = ora.insert_batch(*rec, nthreads=2)
    gsid = [store.new_session() for _ in range(n_sess)]
    g_sids = np.array([gsid[s] for s in sids], np.int32)
    # split into 3 record calls to exercise cross-call state
    cuts = [0, n_ins // 3, 2 * n_ins // 3, n_ins]
    for a, b in zip(cuts[:-1], cuts[1:]):
        sub = pack_records(g_sids[a:b], seqs[a:b], origins[a:b], versions[a:b])
        r = store.record_packed(sub[0], sub[1], sub[2][:-1], np.diff(sub[2]), *sub[3:])
        assert np.array_equal(r.matched, om[a:b])
        assert np.array_equal(r.local, orow[a:b])
        assert np.array_equal(r.parent_local, opar[a:b])
        assert np.array_equal(r.added, oadd[a:b])
    for s in range(n_sess):
        stored, naive, nrows = store.session_stats(gsid[s])
        assert (stored, naive, nrows) == ora.stats(s)
        lex_local = [store.row_info(int(g))["local"] for g in store.session_rows(gsid[s], "lex")]
        assert lex_local == ora.lex_rows(s).tolist()
        rows = store.session_rows(gsid[s], "insert")
        p = store.export(rows)
        for k in range(nrows):
            t, m, v = ora.export_row(s, k)
            a, b = p.offsets[k], p.offsets[k + 1]
            assert np.array_equal(p.tokens[a:b], t)
            assert np.array_equal(p.loss_mask[a:b], m)
            assert np.array_equal(p.versions[a:b], v)
            zeros = np.flatnonzero(m == 0)
            assert p.resp_start[k] == (zeros[-1] + 1 if len(zeros) else 0)
    # read-only matches of fresh queries (host path)
    q = _random_sessions(rng, n_sess, 300, vocab, max_new)
    qsid = np.array([gsid[s] for s in q[0]], np.int32)
    qp = pack_records(q[0], q[1], q[2], q[3])
    m_o, p_o, d_o = ora.match_batch(qp[0], qp[1], qp[2])
    qg = pack_records(qsid, q[1], q[2], q[3])
    m_g, p_g, d_g = store.match(qg[0], qg[1], qg[2][:-1], np.diff(qg[2]))
    assert np.array_equal(m_g, m_o)
    par_local = np.array([store.row_info(int(x))["local"] if x >= 0 else -1 for x in p_g])
    assert np.array_equal(par_local, p_o)
    dup_local = np.array([store.row_info(int(x))["local"] if x >= 0 else -1 for x in d_g])
    assert np.array_equal(dup_local, d_o)


def test_export_deep_chains_and_straddled_tiles(store):
    """K3 corner cases against the C oracle: chains with more ancestor pieces inside one
    4096-position tile than the planner records (in-kernel walk), pieces whose
    boundaries straddle 16-byte output slots, rows spanning several tiles, and output
    offsets of every residue mod 4 (rows exported after a ragged-length row)."""
    rng = np.random.default_rng(2508)
    seqs = []
    cur = rng.integers(0, 151936, 3).tolist()
    for k in range(70):                          # 70-deep chain, 1-7 new tokens per step
        cur = cur + rng.integers(0, 151936, int(rng.integers(1, 8))).tolist()
        seqs.append(list(cur))
        if k % 9 == 4:                           # side branches off the chain
            cut = int(rng.integers(1, len(cur)))
            seqs.append(cur[:cut] + rng.integers(0, 151936, int(rng.integers(1, 6))).tolist())
    long = cur + rng.integers(0, 151936, 9001).tolist()     # multi-tile row on top of the chain
    seqs.append(long)
    seqs.append(long + rng.integers(0, 151936, 5).tolist())
    seqs.append(long[:5000] + rng.integers(0, 151936, 4100).tolist())
    origins = [(rng.random(len(q)) < 0.4).astype(int).tolist() for q in seqs]
    versions = [np.sort(rng.integers(0, 4, len(q))).tolist() for q in seqs]
    ora = CRadixStore()
    ora.insert_batch(*pack_records([0] * len(seqs), seqs, origins, versions))
    sid = store.new_session()
    rec = pack_records([sid] * len(seqs), seqs, origins, versions)
    store.record_packed(rec[0], rec[1], rec[2][:-1], np.diff(rec[2]), *rec[3:])
    rows = np.asarray(store.session_rows(sid, "insert"))
    nrows = len(rows)
    expect = [ora.export_row(0, k) for k in range(nrows)]
    for shift in range(4):  # a ragged row first puts every following row at offset residue `shift`
        order = rng.permutation(nrows)
        head = [k for k in range(nrows) if len(expect[k][0]) % 4 == shift][:1]
        sel = head + order.tolist()
        p = store.export(rows[sel])
        for j, k in enumerate(sel):
            a, b = p.offsets[j], p.offsets[j + 1]
            t, m, v = expect[k]
            assert np.array_equal(p.tokens[a:b], t), (shift, k)
            assert np.array_equal(p.loss_mask[a:b], m), (shift, k)
            assert np.array_equal(p.versions[a:b], v), (shift, k)
            zeros = np.flatnonzero(m == 0)
            assert p.resp_start[j] == (zeros[-1] + 1 if len(zeros) else 0)


def test_long_turn_chains_with_session_path_copies(store):
    """Turn-by-turn sessions deep enough for session path copies (kPathCopyDepth): pure
    extensions (the copy grows in place and is reallocated), branches off every depth
    (the copy moves), re-recorded turns, prefix and diverging queries - all against the
    C oracle, in one batch and across calls, with read-only matches and exports."""
    rng = np.random.default_rng(77)
    n_sess, turns = 6, 90
    sids, seqs = [], []
    cur = {s: [] for s in range(n_sess)}
    hist = {s: [] for s in range(n_sess)}
    for t in range(turns):
        for s in range(n_sess):
            r = rng.random()
            if r < 0.12 and len(hist[s]) > 3:      # branch off an older turn
                base = hist[s][int(rng.integers(len(hist[s])))]
                cut = int(rng.integers(1, len(base)))
                seq = base[:cut] + rng.integers(0, 50, int(rng.integers(1, 40))).tolist()
            elif r < 0.18 and hist[s]:             # re-record an earlier turn
                seq = list(hist[s][int(rng.integers(len(hist[s])))])
            else:                                   # extend the newest turn
                seq = cur[s] + rng.integers(0, 50, int(rng.integers(1, 70))).tolist()
            cur[s] = seq
            hist[s].append(seq)
            sids.append(s)
            seqs.append(seq)
    origins = [(rng.random(len(q)) < 0.5).astype(int).tolist() for q in seqs]
    versions = [np.sort(rng.integers(0, 3, len(q))).tolist() for q in seqs]
    ora = CRadixStore()
    om, orow, opar, oadd = ora.insert_batch(*pack_records(sids, seqs, origins, versions))
    gsid = [store.new_session() for _ in range(n_sess)]
    g_sids = np.array([gsid[s] for s in sids], np.int32)
    cuts = [0, 1, 37, 200, len(seqs)]  # a 1-entry call, then batches of many chained turns
    for a, b in zip(cuts[:-1], cuts[1:]):
        sub = pack_records(g_sids[a:b], seqs[a:b], origins[a:b], versions[a:b])
        r = store.record_packed(sub[0], sub[1], sub[2][:-1], np.diff(sub[2]), *sub[3:])
        assert np.array_equal(r.matched, om[a:b]) and np.array_equal(r.local, orow[a:b])
        assert np.array_equal(r.parent_local, opar[a:b]) and np.array_equal(r.added, oadd[a:b])
    for s in range(n_sess):
        assert store.session_stats(gsid[s]) == ora.stats(s)
        rows = store.session_rows(gsid[s], "insert")
        p = store.export(rows)
        for k in range(len(rows)):
            t, m, v = ora.export_row(s, k)
            a, b = p.offsets[k], p.offsets[k + 1]
            assert np.array_equal(p.tokens[a:b], t) and np.array_equal(p.loss_mask[a:b], m)
            assert np.array_equal(p.versions[a:b], v)
    # read-only queries: prefixes of deep turns, extensions, divergence at every depth
    qs, qsid = [], []
    for _ in range(400):
        s = int(rng.integers(n_sess))
        base = hist[s][int(rng.integers(len(hist[s])))]
        kind = rng.random()
        if kind < 0.3:
            q = base[: int(rng.integers(1, len(base) + 1))]
        elif kind < 0.6:
            q = base + rng.integers(0, 50, int(rng.integers(1, 30))).tolist()
        else:
            cut = int(rng.integers(0, len(base)))
            q = base[:cut] + [int(base[cut]) + 1] + rng.integers(0, 50, 5).tolist()
        qs.append(q)
        qsid.append(s)
    zeros = [[0] * len(q) for q in qs]
    qp = pack_records(qsid, qs, zeros, zeros)
    m_o, p_o, d_o = ora.match_batch(qp[0], qp[1], qp[2])
    qg = pack_records([gsid[s] for s in qsid], qs, zeros, zeros)
    m_g, p_g, d_g = store.match(qg[0], qg[1], qg[2][:-1], np.diff(qg[2]))
    assert np.array_equal(m_g, m_o)
    assert [store.row_info(int(x))["local"] if x >= 0 else -1 for x in p_g] == p_o.tolist()
    assert [store.row_info(int(x))["local"] if x >= 0 else -1 for x in d_g] == d_o.tolist()


def test_device_match_path_and_alignment(store):
    """TM_MEM_DEVICE match on torch tensors equals the host-path result."""
    import torch

    rng = np.random.default_rng(3)
    sid = store.new_session()
    hist = rng.integers(0, 151936, 5000).tolist()
    store.record([sid], [hist], [(np.array([0]), np.array([1], np.uint8), np.array([0]))])
    queries = [hist + [1, 2, 3], hist[:1234] + [int(hist[1234]) + 1], hist[:77], hist, [int(hist[0]) + 1]]
    qp = pack_records([sid] * len(queries), queries, [[0] * len(x) for x in queries], [[0] * len(x) for x in queries], align=32)
    m_h, p_h, d_h = store.match(qp[0], qp[1], qp[2][:-1], np.array([len(x) for x in queries]))
    dev = torch.device("cuda", 0)
    t_sid = torch.from_numpy(qp[0]).to(dev)
    t_tok = torch.from_numpy(qp[1]).to(dev)
    t_off = torch.from_numpy(qp[2][:-1].copy()).to(dev)
    t_len = torch.tensor([len(x) for x in queries], dtype=torch.int64, device=dev)
    om = torch.empty(len(queries), dtype=torch.int64, device=dev)
    op = torch.empty_like(om)
    od = torch.empty_like(om)
    store.match_device(t_sid, t_tok, t_off, t_len, om, op, od)
    torch.cuda.synchronize()
    assert om.cpu().tolist() == m_h.tolist() == [5000, 1234, 77, 5000, 0]
    assert op.cpu().tolist() == p_h.tolist()
    assert od.cpu().tolist() == d_h.tolist()
    assert d_h[3] >= 0 and d_h[0] == -1


def test_errors_map_to_reference_exceptions(store):
    from paper_2508_11553_b200 import SessionTrie

    trie = SessionTrie("err", store=store)
    with pytest.raises(ValueError):
        trie.lpm_insert([], [], [])
    with pytest.raises(ValueError):
        trie.lpm_insert([1, 2], [], [0, 0])
    with pytest.raises(KeyError):
        trie.path_trajectory(5)
    with pytest.raises(KeyError):
        store.session_stats(10**6)


def test_concurrent_threads_match_oracle(store):
    """Many Python threads recording and matching at once (the FastAPI threadpool /
    WorkerPool pattern, trajectory.py:231): per-session results equal the oracle's and a
    session shared by several threads holds exactly the distinct prefixes."""
    import threading

    from paper_2508_11553_b200 import SessionTrie, SpanOrigin, TrajectoryManager

    rng = np.random.default_rng(11)
    n_threads, per = 8, 40
    work = []
    for t in range(n_threads):
        sids, seqs, origins, versions = _random_sessions(np.random.default_rng(100 + t), 3, per, 50, 120)
        work.append((sids, seqs, origins, versions))
    tries = [[SessionTrie(f"t{t}-s{s}", store=store) for s in range(3)] for t in range(n_threads)]
    got = [[None] * per for _ in range(n_threads)]
    tm = TrajectoryManager(type("E", (), {"current_version": 0})(), store=store)
    shared_seqs = [[int(x) for x in rng.integers(0, 30, int(rng.integers(1, 60)))] for _ in range(n_threads * 10)]

    def run(t):
        sids, seqs, origins, versions = work[t]
        for k in range(per):
            org = [SpanOrigin.MODEL_OUTPUT if o else SpanOrigin.AGENT_INPUT for o in origins[k]]
            r = tries[t][sids[k]].lpm_insert(seqs[k], org, versions[k], f"c{k}")
            got[t][k] = (r.matched_prefix_length, r.node_id, r.added_tokens)
            if k % 4 == 0:  # interleave shared-session records through the manager
                for s in shared_seqs[t * 10: t * 10 + 3]:
                    tm.record("shared", s[: max(1, len(s) // 2)], s[max(1, len(s) // 2):], [0] * (len(s) - max(1, len(s) // 2)), 0, f"r{t}-{k}")

    ths = [threading.Thread(target=run, args=(t,)) for t in range(n_threads)]
    [th.start() for th in ths]
    [th.join() for th in ths]
    for t in range(n_threads):
        sids, seqs, origins, versions = work[t]
        ora = CRadixStore()
        om, orow, opar, oadd = ora.insert_batch(*pack_records(sids, seqs, origins, versions))
        assert got[t] == list(zip(om.tolist(), orow.tolist(), oadd.tolist()))
    recorded = []
    for t in range(n_threads):
        for k in range(0, per, 4):
            recorded += [tuple(s) for s in shared_seqs[t * 10: t * 10 + 3]]
    st = tm.storage_stats("shared")
    assert st.stored_tokens == len({q[:i] for q in recorded for i in range(1, len(q) + 1)})
    assert st.naive_tokens == sum(len(q) for q in recorded)
    assert tm.trie_for("shared").check_well_formed() == []


def test_edge_cases_long_sequences_and_extremes(store):
    """Maximum-ish sizes and extreme values: a 1M-token history with a branch at its last
    position, int32-extreme token ids, a batch of 2,000 identical inserts, a query equal to
    a strict prefix, and out-of-range token ids rejected with ValueError."""
    from paper_2508_11553_b200 import SessionTrie, SpanOrigin

    rng = np.random.default_rng(5)
    trie = SessionTrie("long", store=store)
    L = 1 << 20
    h = rng.integers(-(2**31), 2**31 - 1, L, dtype=np.int64).astype(np.int32)
    h[:4] = [-(2**31), 2**31 - 1, 0, -1]
    ins = lambda toks, c: trie.lpm_insert(toks, [SpanOrigin.MODEL_OUTPUT] * len(toks), [7] * len(toks), c)  # noqa: E731
    r0 = ins(h, "a")
    assert (r0.matched_prefix_length, r0.added_tokens) == (0, L)
    b = h.copy()
    b[-1] ^= 1
    r1 = ins(b, "b")
    assert (r1.matched_prefix_length, r1.added_tokens) == (L - 1, 1)
    r2 = ins(h[: L // 2], "c")
    assert (r2.matched_prefix_length, r2.added_tokens) == (L // 2, 0)
    assert trie.stats().stored_tokens == L + 1
    t = trie.path_trajectory(r1.node_id)
    assert t.tokens == b.tolist() and t.version_tags == [7] * L
    m, p, d = store.match([trie.sid], h, [0], [L])
    assert m[0] == L and d[0] == trie.row_of(r0.node_id)
    # 2,000 identical inserts in one batch: one row, naive counts all of them
    sid = store.new_session()
    seq = rng.integers(0, 100, 300).tolist()
    res = store.record([sid] * 2000, [seq] * 2000, [(np.array([0]), np.array([1], np.uint8), np.array([0]))] * 2000)
    assert res.local.tolist() == [0] * 2000 and res.added.tolist() == [300] + [0] * 1999
    assert store.session_stats(sid) == (300, 600_000, 1)
    with pytest.raises(ValueError):
        trie.lpm_insert([2**31], [SpanOrigin.AGENT_INPUT], [0])


def test_pinned_export_views_match_pageable(store):
    """export(pinned=True) / export_ndjson(pinned=True) write the store's page-locked pool
    directly (large results skip the pinned->pageable pass) and equal the pageable path."""
    rng = np.random.default_rng(21)
    sid = store.new_session()
    seqs = [rng.integers(0, 151936, 3_000_000).tolist()] + [rng.integers(0, 151936, 700).tolist() for _ in range(3)]
    runs = [(np.array([0, 5], np.int32), np.array([0, 1], np.uint8), np.array([2, 3], np.int32))] * len(seqs)
    r = store.record([sid] * len(seqs), seqs, runs)
    rows = list(r.row) * 3
    a = store.export(rows)
    b = store.export(rows, pinned=True)
    for x, y in ((a.tokens, b.tokens), (a.loss_mask, b.loss_mask), (a.versions, b.versions), (a.resp_start, b.resp_start)):
        assert np.array_equal(x, y)
    assert np.array_equal(a.offsets, b.offsets)
    names = ["s"] * len(rows)
    assert store.export_ndjson(rows, names) == store.export_ndjson(rows, names, as_array=True, pinned=True).tobytes()


def test_large_host_exports_stream_through_pinned_chunks(store):
    """Exports and NDJSON larger than the single-copy limit (8 MB) come back through the
    chunked pinned pipeline (several chunks, odd sizes); every byte must match."""
    from paper_2508_11553_b200 import Trajectory, trajectory_to_line

    rng = np.random.default_rng(9)
    sid = store.new_session()
    L = (5 << 20) + 12345  # 20 MB of tokens: several 64 MB-or-less chunks across the three arrays
    h = rng.integers(0, 151936, L).astype(np.int32)
    org = (np.arange(L) // 100_000 % 2).astype(np.uint8)
    ver = (np.arange(L) // 1_000_000).astype(np.int32)
    starts = np.flatnonzero(np.r_[True, (org[1:] != org[:-1]) | (ver[1:] != ver[:-1])])
    r = store.record_one(sid, h, (starts.astype(np.int32), org[starts], ver[starts]))
    row = int(r.row[0])
    p = store.export([row, row])
    for k in range(2):
        a, b = p.offsets[k], p.offsets[k + 1]
        assert np.array_equal(p.tokens[a:b], h) and np.array_equal(p.loss_mask[a:b], org)
        assert np.array_equal(p.versions[a:b], ver)
    text = store.export_ndjson([row], ["s-large"])
    t = Trajectory.from_packed("s-large", h, org, ver)
    assert text == (trajectory_to_line(t) + "\n").encode()


def test_hypothesis_naive_oracle_property(store):
    """pkg/tests/test_trie.py:148-174 on the GPU trie: matched == max LCP (the NaiveStore
    oracle), storage == distinct prefixes, every sequence reconstructible, well formed."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    from paper_2508_11553_b200 import SessionTrie, SpanOrigin

    seqs_st = st.lists(st.lists(st.integers(0, 5), min_size=1, max_size=12), min_size=1, max_size=25)

    @given(seqs=seqs_st)
    @settings(max_examples=120, deadline=None)
    def prop(seqs):
        trie = SessionTrie("h", store=store)
        seen = []
        for n, seq in enumerate(seqs):
            want = max([next((i for i, (a, b) in enumerate(zip(s, seq)) if a != b), min(len(s), len(seq)))
                        for s in seen] or [0])
            r = trie.lpm_insert(seq, [SpanOrigin.MODEL_OUTPUT] * len(seq), [0] * len(seq), f"c{n}")
            assert r.matched_prefix_length == want
            seen.append(tuple(seq))
        st_ = trie.stats()
        assert st_.stored_tokens == len({s[:i] for s in seen for i in range(1, len(s) + 1)})
        assert st_.naive_tokens == sum(map(len, seen))
        assert {tuple(t.tokens) for _, t in trie.extract()} == set(seen)
        assert trie.check_well_formed() == []

    prop()


def test_cabi_error_paths(store, tmp_path):
    """Every C-ABI failure is a status code mapped to the reference exception type; the
    store stays usable afterwards."""
    import ctypes as C

    import torch

    from paper_2508_11553_b200 import DeviceStore
    from paper_2508_11553_b200._lib import check

    lib = store.lib
    sid = store.new_session()
    one = (np.array([0], np.int32), np.array([1], np.uint8), np.array([0], np.int32))
    with pytest.raises(KeyError):  # unknown session
        store.record([sid + 10_000], [[1, 2]], [one])
    with pytest.raises(ValueError):  # runs not starting at 0
        store.record([sid], [[1, 2]], [(np.array([1], np.int32), one[1], one[2])])
    with pytest.raises(ValueError):  # run start beyond the sequence
        store.record([sid], [[1, 2]], [(np.array([0, 5], np.int32), np.array([0, 1], np.uint8), np.array([0, 0], np.int32))])
    with pytest.raises(ValueError):  # bad origin code
        store.record([sid], [[1, 2]], [(one[0], np.array([3], np.uint8), one[2])])
    with pytest.raises(KeyError):  # export of a row that does not exist
        store.export([10**9])
    with pytest.raises(KeyError):
        store.row_info(-1)
    dev = torch.device("cuda", 0)
    tok = torch.arange(64, dtype=torch.int32, device=dev)
    with pytest.raises(ValueError):  # device tokens must start on 128-byte boundaries
        store.record_device([sid], tok, [3], [10], [0, 1], *one)
    with pytest.raises(KeyError):  # snapshot that does not exist
        DeviceStore.load(str(tmp_path / "missing"))
    bad = tmp_path / "bad.snap"
    bad.write_bytes(b"NOTASNAPSHOT" * 4)
    with pytest.raises(ValueError):
        DeviceStore.load(str(bad))
    h = C.c_void_p()
    assert lib.tm_store_create(None, None) != 0  # null out pointer
    # still healthy
    r = store.record([sid], [[5, 6, 7]], [one])
    assert r.added.tolist() == [3]


def test_growth_from_tiny_capacities_vs_oracle():
    """Every table starts tiny (arena 64 K words, 64 rows / runs, 16 sessions, 1 K-slot
    branch index) and grows — arena and row-table reallocation, branch-index rehash, dense
    probe collisions — with results still equal to the oracle's."""
    from paper_2508_11553_b200 import DeviceStore

    st = DeviceStore(0, arena_words=1 << 16, row_capacity=64, run_capacity=64, session_capacity=16)
    rng = np.random.default_rng(99)
    n_sess = 300
    sids, seqs, origins, versions = _random_sessions(rng, n_sess, 3000, 151936, 400)
    g = [st.new_session() for _ in range(n_sess)]
    ora = CRadixStore()
    om, orow, opar, oadd = ora.insert_batch(*pack_records(sids, seqs, origins, versions), nthreads=4)
    for a in range(0, len(sids), 700):  # several calls, each forcing growth
        b = min(len(sids), a + 700)
        sub = pack_records([g[s] for s in sids[a:b]], seqs[a:b], origins[a:b], versions[a:b])
        r = st.record_packed(sub[0], sub[1], sub[2][:-1], np.diff(sub[2]), *sub[3:])
        assert np.array_equal(r.matched, om[a:b]) and np.array_equal(r.local, orow[a:b])
        assert np.array_equal(r.parent_local, opar[a:b])
    info = st.stats()
    assert info["arena_cap"] > (1 << 16) and info["rows"] == sum(ora.stats(s)[2] for s in range(n_sess))
    for s in (0, 17, 299):
        rows = st.session_rows(g[s])
        p = st.export(rows)
        for k in range(len(rows)):
            t, m, v = ora.export_row(s, k)
            assert np.array_equal(p.tokens[p.offsets[k]:p.offsets[k + 1]], t)
    st.close()
