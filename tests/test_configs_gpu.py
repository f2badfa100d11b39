"""Configs 1-3 of BASELINE.json through the B200 store: bit-exact against the C
oracle at reduced session counts, and at full size through size-independent
properties (closed-form storage, matched lengths, export == what was recorded with
first-writer metadata)."""

import numpy as np
import pytest

from oracle.cport import CRadixStore
from workloads import RecordWorkload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def store():
    from paper_2508_11553_b200 import DeviceStore

    s = DeviceStore(0)
    yield s
    s.close()


def _record(store, wl):
    sid_map = [store.new_session() for _ in range(wl.n_sessions)]
    sids, tok, off, roff, rs, ro, rv = wl.packed(sid_map)
    res = store.record_packed(sids, tok, off[:-1], np.diff(off), roff, rs, ro, rv)
    return sid_map, res


@pytest.mark.parametrize("config,n", [(1, 3), (2, 20), (3, 200)])
def test_config_vs_c_oracle(store, config, n):
    wl = RecordWorkload(config, n_sessions=n)
    ora = CRadixStore()
    om, orow, opar, oadd = ora.insert_batch(*wl.packed(), nthreads=4)
    sid_map, r = _record(store, wl)
    assert np.array_equal(r.matched, om) and np.array_equal(r.local, orow)
    assert np.array_equal(r.parent_local, opar) and np.array_equal(r.added, oadd)
    for s in range(n):
        assert store.session_stats(sid_map[s]) == ora.stats(s)
        rows = store.session_rows(sid_map[s], "lex")
        p = store.export(rows)
        lex = ora.lex_rows(s)
        assert [store.row_info(int(g))["local"] for g in rows] == lex.tolist()
        for i, k in enumerate(lex):
            t, m, v = ora.export_row(s, int(k))
            a, b = p.offsets[i], p.offsets[i + 1]
            assert np.array_equal(p.tokens[a:b], t) and np.array_equal(p.loss_mask[a:b], m)
            assert np.array_equal(p.versions[a:b], v)


def test_config2_full_size_closed_form(store):
    """1,000 sessions x 16 branches x 8,192 tokens: stored = P + 16 S per session,
    matched = P for branches 1..15, every exported row == its recorded tokens."""
    wl = RecordWorkload(2)
    sid_map, r = _record(store, wl)
    P, S, K = 6144, 2048, 16
    m = r.matched.reshape(-1, K)
    assert np.all(m[:, 0] == 0) and np.all(m[:, 1:] == P)
    assert np.all(r.parent_local.reshape(-1, K)[:, 1:] == 0)
    for s in (0, 499, 999):
        assert store.session_stats(sid_map[s])[:2] == (P + K * S, K * (P + S))
    p = store.export(r.row)
    lens = np.diff(p.offsets)
    assert np.all(lens == P + S)
    toks = p.tokens.reshape(-1, P + S)
    want = np.stack(wl.seqs)
    assert np.array_equal(toks, want)
    mask = p.loss_mask.reshape(-1, P + S)
    assert not mask[:, : P + 512].any() and mask[:, P + 512:].all()
    assert np.all(p.resp_start == P + 512)


def test_config3_full_size_stitch(store):
    """4,000 sessions: turn 2 keeps turn 1's first-writer metadata for positions < 2,048
    and the stitched legs' versions (v0 then v1 at the split) after."""
    wl = RecordWorkload(3)
    sid_map, r = _record(store, wl)
    assert np.all(r.matched[0::2] == 0) and np.all(r.matched[1::2] == 2048)
    p = store.export(r.row[1::2])
    L = 2048 + 512 + 1536
    toks = p.tokens.reshape(-1, L)
    assert np.array_equal(toks, np.stack(wl.seqs[1::2]))
    mask = p.loss_mask.reshape(-1, L)
    vers = p.versions.reshape(-1, L)
    assert not mask[:, :1024].any() and mask[:, 1024:2048].all() and not mask[:, 2048:2560].any()
    assert mask[:, 2560:].all()
    split = np.array(wl.split)
    pos = np.arange(L)[None, :]
    want_v = np.where(pos >= 2560 + split[:, None], 1, 0)
    assert np.array_equal(vers, want_v)
    assert np.all(p.resp_start == 2560)


def test_config1_turns(store):
    wl = RecordWorkload(1)
    sid_map, r = _record(store, wl)
    assert r.matched.tolist() == [0] + [512 * t for t in range(1, 8)]
    assert r.parent_local.tolist() == [-1] + list(range(7))
    rows = store.session_rows(sid_map[0], "lex")
    p = store.export(rows)
    assert [int(x) for x in np.diff(p.offsets)] == [512 * (t + 1) for t in range(8)]
    full = p.tokens[p.offsets[7]: p.offsets[8]]
    assert np.array_equal(full, wl.seqs[7])
    v = p.versions[p.offsets[7]: p.offsets[8]]
    # first-writer: turn t's tokens carry turn t's version (bump from turn 5)
    assert np.array_equal(v, np.repeat([0, 0, 0, 0, 0, 1, 1, 1], 512))
