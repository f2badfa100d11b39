"""Full-size parity on BASELINE.json's configs (not reduced session counts): every value the
B200 store returns is compared with the C restatement of the reference trie
(oracle/radix_oracle.c, itself pinned to the reference's golden vectors) — and, for the
include_partials export of config 3, with the UNMODIFIED reference's own
TrajectoryManager._partial_trajectory / extract_trajectories (trajectory.py:299-340)
imported from baseline/_ref.

  c2  1,000 sessions x 16 branches x 8,192 tokens (16,000 records, 131 M tokens):
      matched / node id / parent / added of every record, StorageStats of every session,
      lexicographic extract order of every session, and every exported token / loss-mask /
      version of all 16,000 rows
  c3  4,000 sessions x 2 turns (stitched v0/v1 legs): the same, all 8,000 rows; then 10 %
      of the sessions left paused mid-turn-2 and exported with include_partials
  c4  10,000 sessions x 32,768 tokens, one 4,096-query batch: matched, parent and
      duplicate row of every query (the bench checks matched lengths only)
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from oracle.cport import CRadixStore
from workloads import MatchWorkload, RecordWorkload

pytestmark = pytest.mark.gpu
NTHREADS = os.cpu_count() or 4
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture
def store():
    from paper_2508_11553_b200 import DeviceStore

    s = DeviceStore(0)
    yield s
    s.close()


def _record_both(store, wl):
    ora = CRadixStore()
    om, orow, opar, oadd = ora.insert_batch(*wl.packed(), nthreads=NTHREADS)
    sid_map = [store.new_session() for _ in range(wl.n_sessions)]
    sids, tok, off, roff, rs, ro, rv = wl.packed(sid_map)
    r = store.record_packed(sids, tok, off[:-1], np.diff(off), roff, rs, ro, rv)
    return ora, sid_map, (om, orow, opar, oadd), r


def _check_records_and_exports(store, wl, ora, sid_map, o, r):
    om, orow, opar, oadd = o
    assert np.array_equal(r.matched, om), "matched_prefix_length"
    assert np.array_equal(r.local, orow), "node id"
    assert np.array_equal(r.parent_local, opar), "chosen parent"
    assert np.array_equal(r.added, oadd), "added_tokens"
    rows_g, sess_o, rows_o = [], [], []
    for s in range(wl.n_sessions):
        assert store.session_stats(sid_map[s]) == ora.stats(s), f"StorageStats of session {s}"
        lex_g = store.session_rows(sid_map[s], "lex")
        lex_o = ora.lex_rows(s)
        rows_g.append(lex_g)
        sess_o.append(np.full(len(lex_o), s, np.int64))
        rows_o.append(lex_o)
    rows_g = np.concatenate(rows_g)
    loc_g = np.array([store.row_info(int(g))["local"] for g in rows_g])
    assert np.array_equal(loc_g, np.concatenate(rows_o)), "extract (lexicographic) order"
    p = store.export(rows_g)
    off, t, m, v = ora.export_batch(np.concatenate(sess_o), np.concatenate(rows_o), nthreads=NTHREADS)
    assert np.array_equal(p.offsets, off)
    assert np.array_equal(p.tokens, t), "exported tokens"
    assert np.array_equal(p.loss_mask, m), "exported loss_mask"
    assert np.array_equal(p.versions, v), "exported versions"
    return p


def test_config2_full_size_vs_oracle(store):
    wl = RecordWorkload(2)
    ora, sid_map, o, r = _record_both(store, wl)
    p = _check_records_and_exports(store, wl, ora, sid_map, o, r)
    assert len(p.offsets) == 16_001 and p.offsets[-1] == 16_000 * 8192


def test_config3_full_size_vs_oracle(store):
    wl = RecordWorkload(3)
    ora, sid_map, o, r = _record_both(store, wl)
    p = _check_records_and_exports(store, wl, ora, sid_map, o, r)
    assert len(p.offsets) == 8_001


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "rolloutlab")), reason="baseline/_ref not installed")
def test_config3_include_partials_vs_reference(store):
    """c3 with 10 % of the sessions paused inside turn 2 (after the first leg, or inside
    the second): extract_trajectories(include_partials=True) of the drop-in manager vs the
    unmodified reference manager holding the same completed records and the same open
    requests.  Completed rows come from the GPU export; partials follow trajectory.py:329-340."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rolloutlab.trajectory as RT  # the reference, unaliased (this process never installs refalias)

    from paper_2508_11553_b200 import GenParams, TrajectoryManager
    from paper_2508_11553_b200.trajectory import PendingRequest

    assert RT.__file__.startswith(REF), RT.__file__
    wl = RecordWorkload(3)
    n = wl.n_sessions
    rng = np.random.default_rng(20251021)
    paused = set(rng.choice(n, n // 10, replace=False).tolist())

    class _Engine:  # only current_version is read when requests open
        current_version = 0

    tm = TrajectoryManager(_Engine(), store=store)
    ref = RT.TrajectoryManager(_Engine())
    recs = []
    for s in range(n):
        t1 = wl.seqs[2 * s]
        recs.append(dict(session_id=f"c3-{s}", input_tokens=t1[:1024].tolist(), produced=t1[1024:].tolist(),
                         versions=[0] * 1024, context_version=0, request_id=f"r{s}-1"))
        if s not in paused:
            t2 = wl.seqs[2 * s + 1]
            k = wl.split[s]
            recs.append(dict(session_id=f"c3-{s}", input_tokens=t2[:2560].tolist(), produced=t2[2560:].tolist(),
                             versions=[0] * k + [1] * (1536 - k), context_version=0, request_id=f"r{s}-2"))
    tm.record_many(recs)
    # the same completed exchanges through the reference's own recording path
    for rec in recs:
        if int(rec["session_id"].split("-")[1]) not in paused:
            continue
        req = RT.PendingRequest(request_id=rec["request_id"], session_id=rec["session_id"],
                                input_tokens=rec["input_tokens"], params=RT.GenParams(max_new_tokens=4096),
                                context_version=0)
        req.produced, req.versions = list(rec["produced"]), list(rec["versions"])
        ref._session(rec["session_id"], create=True)
        ref._open_requests[req.request_id] = req
        ref._finalize(req)
    # open (paused) turn-2 requests: the first leg only, or both legs cut inside leg 2
    for s in sorted(paused):
        t2 = wl.seqs[2 * s + 1]
        k = wl.split[s]
        cut = k if s % 2 else k + int(rng.integers(1, 1536 - k + 1))
        produced = t2[2560: 2560 + cut].tolist()
        versions = [0] * min(cut, k) + [1] * max(0, cut - k)
        for mgr, Req, Par in ((tm, PendingRequest, GenParams), (ref, RT.PendingRequest, RT.GenParams)):
            req = Req(request_id=f"r{s}-2", session_id=f"c3-{s}", input_tokens=t2[:2560].tolist(),
                      params=Par(max_new_tokens=1536), context_version=0)
            req.produced, req.versions = produced, versions
            mgr._open_requests[req.request_id] = req
    n_partial = 0
    for s in sorted(paused):
        sid = f"c3-{s}"
        got = tm.extract_trajectories(sid, include_partials=True)
        exp = ref.extract_trajectories(sid, include_partials=True)
        assert len(got) == len(exp) == 2
        for g, e in zip(got, exp):
            assert g.session_id == e.session_id
            assert g.tokens == e.tokens and g.loss_mask == e.loss_mask and g.version_tags == e.version_tags
        n_partial += 1
        for mv in (1,):
            g1 = tm.extract_trajectories(sid, include_partials=True, min_version=mv)
            e1 = ref.extract_trajectories(sid, include_partials=True, min_version=mv)
            assert [t.tokens for t in g1] == [t.tokens for t in e1]
    assert n_partial == n // 10
    # the same export in tensor form, assembled on the GPU (completed rows: K3; partials:
    # k_fill_host_rows), against the reference's objects in extract_trajectories order
    names = [f"c3-{s}" for s in sorted(paused)]
    row_sids, packed, order = tm.export_packed(names, include_partials=True)
    exp = [t for sid in names for t in ref.extract_trajectories(sid, include_partials=True)]
    assert len(order) == len(exp) == 2 * len(names)
    off = packed.offsets
    tok = packed.tokens.cpu().numpy()
    msk = packed.loss_mask.cpu().numpy()
    ver = packed.versions.cpu().numpy()
    resp = packed.resp_start.cpu().numpy()
    for i, e in zip(order, exp):
        a, b = off[i], off[i + 1]
        assert row_sids[i] == e.session_id
        assert tok[a:b].tolist() == e.tokens
        assert msk[a:b].astype(bool).tolist() == e.loss_mask
        assert ver[a:b].tolist() == e.version_tags
        assert resp[i] == (max([k for k, x in enumerate(e.loss_mask) if not x], default=-1) + 1)
    # sessions that completed both turns: no partials, two completed rows each
    for s in range(0, n, 97):
        if s in paused:
            continue
        got = tm.extract_trajectories(f"c3-{s}", include_partials=True)
        assert [len(t.tokens) for t in got] == [2048, 4096]


def test_config4_full_batch_parent_and_dup_vs_oracle(store):
    """The bench's c4 batch at full size: matched, parent and duplicate row of all 4,096
    queries against the C oracle (after branching a third of the sessions so parents are
    not trivially the session's only row)."""
    wl = MatchWorkload(10_000, 32_768, 4096)
    ns = wl.n_sessions
    ora = CRadixStore()
    toks = np.concatenate([wl.hist_tokens[wl.hist_off[s]: wl.hist_off[s] + wl.hist_len[s]] for s in range(ns)])
    off = np.zeros(ns + 1, np.int64)
    np.cumsum(wl.hist_len, out=off[1:])
    ora.insert_batch(np.arange(ns, dtype=np.int32), toks, off, wl.run_off, wl.run_start, wl.run_origin,
                     wl.run_version, nthreads=NTHREADS)
    sids = [store.new_session() for _ in range(ns)]
    assert sids == list(range(ns))
    store.record_packed(np.arange(ns, dtype=np.int32), wl.hist_tokens, wl.hist_off[:-1].copy(), wl.hist_len,
                        wl.run_off, wl.run_start, wl.run_origin, wl.run_version)
    # branch every third session of a second query set into both stores
    br = wl.make_queries(np.random.default_rng(5))
    pick = np.arange(0, wl.n_queries, 3)
    bt = [br["q_tokens"][br["q_off"][i]: br["q_off"][i] + br["q_len"][i]] for i in pick]
    bo = np.zeros(len(bt) + 1, np.int64)
    np.cumsum([len(x) for x in bt], out=bo[1:])
    bs = br["q_sess"][pick]
    zr = np.arange(len(bt) + 1, dtype=np.int64)
    z32 = np.zeros(len(bt), np.int32)
    o8 = np.ones(len(bt), np.uint8)
    ora.insert_batch(bs, np.concatenate(bt), bo, zr, z32, o8, z32 + 1, nthreads=NTHREADS)
    store.record_packed(bs, np.concatenate(bt), bo[:-1], np.diff(bo), zr, z32, o8, z32 + 1)
    q = [wl.q_tokens[wl.q_off[i]: wl.q_off[i] + wl.q_len[i]] for i in range(wl.n_queries)]
    qo = np.zeros(len(q) + 1, np.int64)
    np.cumsum([len(x) for x in q], out=qo[1:])
    m_o, p_o, d_o = ora.match_batch(wl.q_sess, np.concatenate(q), qo, nthreads=NTHREADS)
    m_g, p_g, d_g = store.match(wl.q_sess, wl.q_tokens, wl.q_off[:-1].copy(), wl.q_len)
    assert np.array_equal(m_g, m_o)
    loc = lambda rows: np.array([store.row_info(int(x))["local"] if x >= 0 else -1 for x in rows])  # noqa: E731
    assert np.array_equal(loc(p_g), p_o), "parent rows"
    assert np.array_equal(loc(d_g), d_o), "duplicate rows"
    # queries on the branched rows themselves: re-records (dup = the branch), extensions
    # (parent = the branch) and prefixes of them, against the oracle again
    qq, qs = [], []
    for j, x in enumerate(bt):
        kind = j % 3
        qq.append(np.concatenate([x, [7, 8, 9]]) if kind == 0 else (x if kind == 1 else x[: max(1, len(x) - 100)]))
        qs.append(bs[j])
    qo2 = np.zeros(len(qq) + 1, np.int64)
    np.cumsum([len(x) for x in qq], out=qo2[1:])
    qt2 = np.concatenate(qq).astype(np.int32)
    qs = np.asarray(qs, np.int32)
    m_o, p_o, d_o = ora.match_batch(qs, qt2, qo2, nthreads=NTHREADS)
    m_g, p_g, d_g = store.match(qs, qt2, qo2[:-1], np.diff(qo2))
    assert np.array_equal(m_g, m_o)
    assert np.array_equal(loc(p_g), p_o) and np.array_equal(loc(d_g), d_o)
    assert (p_o > 0).any() and (d_o > 0).any(), "queries resolve to branched rows"
