"""Resource bounds and input validation of the store (round-2 review findings):

* sampling many completions of one deep turn (siblings at chain depth >= kPathCopyDepth)
  must not give every sibling a full session path copy: arena use stays within a small
  multiple of the stored tokens, and every value still matches the C oracle;
* re-recording an existing sequence leaves its reserved row id as a hole that the next
  new row reuses (the row table grows with distinct sequences, not with calls);
* device-buffer matches with session ids the store never created return matched 0;
* TrajectoryManager.save() while other threads keep recording: every snapshot's sidecar
  agrees with its store (no row reaches the store without reaching the sidecar).
"""

from __future__ import annotations

import threading

import numpy as np
import pytest

from oracle.cport import CRadixStore
from workloads import pack_records

pytestmark = pytest.mark.gpu


@pytest.fixture
def store():
    from paper_2508_11553_b200 import DeviceStore

    s = DeviceStore(0)
    yield s
    s.close()


def test_deep_siblings_do_not_copy_the_path_each(store):
    rng = np.random.default_rng(11)
    n_sess, turns, samples, L_turn, L_out = 4, 6, 48, 900, 40
    sids, seqs = [], []
    for s in range(n_sess):
        ctx = []
        for _ in range(turns):  # a turn-by-turn chain: depth 0..turns-1 (copies from depth 4)
            ctx = ctx + rng.integers(0, 151936, L_turn).tolist()
            sids.append(s)
            seqs.append(ctx)
        base = ctx + rng.integers(0, 151936, 100).tolist()  # the next turn's input
        for _ in range(samples):  # N sampled completions of that input: siblings at depth `turns`
            sids.append(s)
            seqs.append(base + rng.integers(0, 151936, L_out).tolist())
    origins = [[0] * len(q) for q in seqs]
    versions = [[0] * len(q) for q in seqs]
    ora = CRadixStore()
    om, orow, opar, oadd = ora.insert_batch(*pack_records(sids, seqs, origins, versions))
    gs = [store.new_session() for _ in range(n_sess)]
    packed = pack_records([gs[s] for s in sids], seqs, origins, versions)
    half = len(seqs) // 2  # two calls: siblings recorded in one launch and across launches
    for a, b in ((0, half), (half, len(seqs))):
        sub = pack_records([gs[s] for s in sids[a:b]], seqs[a:b], origins[a:b], versions[a:b])
        r = store.record_packed(sub[0], sub[1], sub[2][:-1], np.diff(sub[2]), *sub[3:])
        assert np.array_equal(r.matched, om[a:b]) and np.array_equal(r.local, orow[a:b])
        assert np.array_equal(r.parent_local, opar[a:b]) and np.array_equal(r.added, oadd[a:b])
    stored = sum(store.session_stats(g)[0] for g in gs)
    assert stored == sum(ora.stats(s)[0] for s in range(n_sess))
    used = store.stats()["arena_used"]
    longest = max(len(q) for q in seqs)
    nrows = store.stats()["rows"]
    # rows (each padded to 128-byte lines) + at most a doubling chain of copies per session
    bound = stored + 64 * nrows + n_sess * 4 * (longest + 64)
    assert used <= bound, (used, bound, stored)
    # the pre-fix behaviour (a fresh 2L copy per sibling) would need far more
    assert used < stored + n_sess * samples * 2 * (turns * L_turn) // 4
    # walks over the siblings still agree with the oracle
    qs = [seqs[k] + [5, 6] for k in range(0, len(seqs), 7)]
    qsid = [sids[k] for k in range(0, len(seqs), 7)]
    z = [[0] * len(q) for q in qs]
    qo = pack_records(qsid, qs, z, z)
    m_o, _, _ = ora.match_batch(qo[0], qo[1], qo[2])
    qg = pack_records([gs[s] for s in qsid], qs, z, z)
    m_g, _, _ = store.match(qg[0], qg[1], qg[2][:-1], np.diff(qg[2]))
    assert np.array_equal(m_g, m_o)
    del packed


def test_rerecorded_sequences_leave_reusable_row_holes(store):
    sid = store.new_session()
    one = (np.array([0], np.int32), np.array([1], np.uint8), np.array([0], np.int32))
    a = list(range(100, 164))
    r0 = store.record([sid], [a], [one])
    row_a = int(r0.row[0])
    r1 = store.record([sid], [a], [one])  # duplicate: reserves the next id, leaves it empty
    assert int(r1.row[0]) == row_a and int(r1.matched[0]) == 64 and int(r1.added[0]) == 0
    for _ in range(5):
        store.record([sid, sid], [a, a], [one, one])  # more duplicates
    r2 = store.record([sid], [a + [7]], [one])
    assert int(r2.row[0]) <= row_a + 2, "the new row reuses a hole instead of a fresh id"
    assert store.stats()["rows"] == 2
    assert store.session_stats(sid) == (65, 64 * 12 + 65, 2)
    p = store.export([int(r2.row[0])])
    assert p.tokens.tolist() == a + [7]
    assert int(r2.local[0]) == 1 and int(r2.parent_local[0]) == 0


def test_device_match_with_unknown_session_ids(store):
    import torch

    sid = store.new_session()
    hist = list(range(1, 300))
    store.record([sid], [hist], [(np.array([0], np.int32), np.array([1], np.uint8), np.array([0], np.int32))])
    bad = [sid, 10**6, -5, sid + 1]
    qs = [hist + [1], hist, hist, hist]
    qp = pack_records(bad, qs, [[0] * len(q) for q in qs], [[0] * len(q) for q in qs], align=32)
    dev = torch.device("cuda", 0)
    om = torch.full((4,), 7, dtype=torch.int64, device=dev)
    op = torch.full_like(om, 7)
    od = torch.full_like(om, 7)
    store.match_device(torch.from_numpy(qp[0]).to(dev), torch.from_numpy(qp[1]).to(dev),
                       torch.from_numpy(qp[2][:-1].copy()).to(dev),
                       torch.tensor([len(q) for q in qs], dtype=torch.int64, device=dev), om, op, od)
    torch.cuda.synchronize()
    assert om.cpu().tolist() == [299, 0, 0, 0]
    assert op.cpu().tolist()[1:] == [-1, -1, -1] and od.cpu().tolist()[1:] == [-1, -1, -1]
    store.synchronize()  # no device error was raised


def test_save_while_recording_keeps_sidecar_and_store_in_step(store, tmp_path):
    from paper_2508_11553_b200 import DeviceStore, TrajectoryManager

    class _Engine:
        current_version = 0

    tm = TrajectoryManager(_Engine(), store=store)
    stop = threading.Event()
    errors = []

    def writer(w):
        rng = np.random.default_rng(w)
        k = 0
        try:
            while not stop.is_set():
                s = f"w{w}-s{k % 5}"
                inp = rng.integers(0, 1000, int(rng.integers(1, 50))).tolist()
                out = rng.integers(0, 1000, int(rng.integers(1, 50))).tolist()
                tm.record(s, inp, out, [0] * len(out), 0, f"w{w}-r{k}")
                k += 1
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=writer, args=(w,)) for w in range(6)]
    for t in threads:
        t.start()
    paths = []
    try:
        for i in range(6):
            p = str(tmp_path / f"snap{i}")
            tm.save(p)
            paths.append(p)
    finally:
        stop.set()
        for t in threads:
            t.join()
    assert not errors, errors
    for p in paths:
        tm2 = TrajectoryManager.load(p, _Engine())
        for sid in tm2.session_ids():
            trie = tm2.trie_for(sid)
            nrows = trie.store.session_stats(trie.sid)[2]
            assert nrows == len(trie._rows), (p, sid, nrows, len(trie._rows))
            assert len(trie.extract()) == len(trie._marks)
        for st in tm2.stores:
            st.close()
    assert DeviceStore  # imported for the loader's type
