"""Packed host->device token copies (csrc/hostpack.cpp + k_unpack18) against the raw
int32 copy, through the C ABI.

Stores are created with TM_H2D_PACK_MIN=0 (every host-memory call is packed) and -1 (never
packed).  Results must be identical to each other and to the C oracle; the h2d counters
prove which path ran, including the fallback for ids outside [0, 2^18).
"""

import os

import numpy as np
import pytest

from oracle.cport import CRadixStore
from workloads import pack_records

pytestmark = pytest.mark.gpu


def _store(pack_min, frac=None):
    from paper_2508_11553_b200 import DeviceStore

    env = {"TM_H2D_PACK_MIN": str(pack_min)}
    if frac is not None:
        env["TM_H2D_PACK_FRAC"] = str(frac)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return DeviceStore(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


def _sessions(rng, n_sess, n_ins, vocab, max_new):
    sids, seqs = [], []
    ctx = {s: [[]] for s in range(n_sess)}
    for _ in range(n_ins):
        s = int(rng.integers(n_sess))
        base = ctx[s][int(rng.integers(len(ctx[s])))]
        if rng.random() < 0.3 and len(base) > 2:
            cut = int(rng.integers(1, len(base)))
            seq = base[:cut] + vocab(rng, int(rng.integers(1, max_new)))
        else:
            seq = base + vocab(rng, int(rng.integers(1, max_new)))
        sids.append(s)
        seqs.append(seq)
        ctx[s].append(seq)
    return sids, seqs


def _small_ids(rng, n):
    return rng.integers(0, 1 << 18, n).tolist()


def _wide_ids(rng, n):  # ids the 18-bit planes cannot carry
    x = rng.integers(0, 151936, n)
    x[rng.random(n) < 0.01] = (1 << 18) + 5
    x[rng.random(n) < 0.01] = 2**31 - 1
    x[rng.random(n) < 0.01] = -7
    return x.tolist()


def _record_and_match(store, sids, seqs, align):
    gs = [store.new_session() for _ in range(max(sids) + 1)]
    org = [[int(i % 3 == 0) for i in range(len(q))] for q in seqs]
    ver = [[0] * len(q) for q in seqs]
    rec = pack_records([gs[s] for s in sids], seqs, org, ver, align=align)
    lens = np.array([len(q) for q in seqs], np.int64)
    tok_off = rec[2][:-1]
    r = store.record_packed(rec[0], rec[1], tok_off, lens, *rec[3:])
    m, p, d = store.match(rec[0], rec[1], tok_off, lens)
    rows = np.concatenate([store.session_rows(g, "insert") for g in gs])
    ex = store.export(rows)
    return r, (m, p, d), ex


@pytest.mark.parametrize("align", [1, 32])
@pytest.mark.parametrize("ids", ["small", "wide"])
def test_packed_copy_equals_raw_copy(align, ids):
    rng = np.random.default_rng(11 + align)
    vocab = _small_ids if ids == "small" else _wide_ids
    sids, seqs = _sessions(rng, 12, 240, vocab, 900)
    packed, raw = _store(0), _store(-1)
    try:
        rp, mp, ep = _record_and_match(packed, sids, seqs, align)
        rr, mr, er = _record_and_match(raw, sids, seqs, align)
        for f in ("matched", "local", "parent_local", "added"):
            assert np.array_equal(getattr(rp, f), getattr(rr, f)), f
        for a, b in zip(mp, mr):
            assert np.array_equal(a, b)
        for f in ("offsets", "tokens", "loss_mask", "versions", "resp_start"):
            assert np.array_equal(getattr(ep, f), getattr(er, f)), f
        hp, hr = packed.h2d_stats(), raw.h2d_stats()
        assert hr["packed_calls"] == 0 and hr["raw_calls"] == 2
        if ids == "small":
            assert hp["packed_calls"] == 2 and hp["pack_fallbacks"] == 0
            assert hp["packed_tokens"] == 2 * sum(len(q) for q in seqs)
        else:
            assert hp["pack_fallbacks"] == 2 and hp["raw_calls"] == 2
        # and against the C oracle
        ora = CRadixStore()
        org = [[int(i % 3 == 0) for i in range(len(q))] for q in seqs]
        om, orow, opar, oadd = ora.insert_batch(*pack_records(sids, seqs, org, [[0] * len(q) for q in seqs]))
        assert np.array_equal(rp.matched, om) and np.array_equal(rp.added, oadd)
    finally:
        packed.close()
        raw.close()


def test_aligned_layout_with_shared_ranges_and_garbage_gaps():
    """Caller buffers with 32-aligned starts: two queries may share words, and the words
    between sequences hold values the planes cannot carry - they are not part of any
    sequence, so they must neither be packed nor force the fallback."""
    rng = np.random.default_rng(5)
    hist = [rng.integers(0, 151936, int(rng.integers(100, 3000))).tolist() for _ in range(6)]
    buf = np.full(40000, -123456789, np.int32)  # garbage everywhere but the sequences
    offs, lens, qsess = [], [], []
    pos = 0
    for k, h in enumerate(hist):
        q = h + rng.integers(0, 151936, 7).tolist() if k % 2 else h[: len(h) // 2]
        buf[pos: pos + len(q)] = q
        offs += [pos, pos]                       # the same words twice, two lengths
        lens += [len(q), max(1, len(q) - 40)]
        qsess += [k, k]
        pos += (len(q) + 31) // 32 * 32 + 64
    packed, raw = _store(0), _store(-1)
    try:
        outs = []
        for st in (packed, raw):
            gs = [st.new_session() for _ in hist]
            rec = pack_records(gs, hist, [[0] * len(h) for h in hist], [[1] * len(h) for h in hist])
            st.record_packed(rec[0], rec[1], rec[2][:-1], np.diff(rec[2]), *rec[3:])
            sids = np.array([gs[k] for k in qsess], np.int32)
            m, p, d = st.match(sids, buf, np.array(offs, np.int64), np.array(lens, np.int64))
            outs.append((m, [st.row_info(int(x))["local"] if x >= 0 else -1 for x in p]))
        assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
        exp = [min(lens[j], len(hist[qsess[j]])) for j in range(len(lens))]
        assert outs[0][0].tolist() == exp
        h = packed.h2d_stats()
        assert h["pack_fallbacks"] == 0 and h["packed_calls"] == 2
    finally:
        packed.close()
        raw.close()


def test_small_calls_stay_raw_by_default():
    from paper_2508_11553_b200 import DeviceStore

    st = DeviceStore(0)
    try:
        s = st.new_session()
        st.record_one(s, np.arange(100, dtype=np.int32),
                      (np.zeros(1, np.int32), np.zeros(1, np.uint8), np.zeros(1, np.int32)))
        h = st.h2d_stats()
        assert h["packed_calls"] == 0 and h["raw_calls"] == 1
    finally:
        st.close()


def test_auto_policy_stays_raw_with_several_gpu_clients():
    """TM_H2D_PACK_MIN unset: packing doubles host-memory traffic, so it is skipped when
    more than one store is live in the process (or LOCAL_WORLD_SIZE > 1)."""
    from paper_2508_11553_b200 import DeviceStore

    assert "TM_H2D_PACK_MIN" not in os.environ
    a, b = DeviceStore(0), DeviceStore(0)
    try:
        s = a.new_session()
        n = 9 << 20  # above the 8M-token default threshold
        toks = (np.arange(n, dtype=np.int64) % 151936).astype(np.int32)
        a.record_one(s, toks, (np.zeros(1, np.int32), np.zeros(1, np.uint8), np.zeros(1, np.int32)))
        h = a.h2d_stats()
        assert h["packed_calls"] == 0 and h["raw_calls"] == 1 and h["token_bytes"] == 4 * n
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("frac", [0.0, 0.37, 0.8])
def test_hybrid_split_packed_head_raw_tail(frac):
    """TM_H2D_PACK_FRAC < 1: the head of an aligned call's token range is packed, the tail
    goes raw from the caller's buffer in the same call; results equal the raw copy's."""
    rng = np.random.default_rng(23)
    sids, seqs = _sessions(rng, 16, 300, _small_ids, 1500)
    hyb, raw = _store(0, frac), _store(-1)
    try:
        rh, mh, eh = _record_and_match(hyb, sids, seqs, 32)
        rr, mr, er = _record_and_match(raw, sids, seqs, 32)
        for f in ("matched", "local", "parent_local", "added"):
            assert np.array_equal(getattr(rh, f), getattr(rr, f)), f
        for a, b in zip(mh, mr):
            assert np.array_equal(a, b)
        for f in ("offsets", "tokens", "loss_mask", "versions", "resp_start"):
            assert np.array_equal(getattr(eh, f), getattr(er, f)), f
        h = hyb.h2d_stats()
        assert h["pack_fallbacks"] == 0 and h["packed_calls"] == 2
        total = 2 * sum(len(q) for q in seqs)
        # fewer PCIe bytes than raw unless nothing is packed
        assert (h["token_bytes"] < 4 * total) == (frac > 0)
    finally:
        hyb.close()
        raw.close()
