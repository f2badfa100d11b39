"""_tmfast (csrc/tmfast.c): the CPython extension that turns the drop-in's Python arguments
into C buffers (token lists -> int32, per-token origins / versions -> metadata runs,
threaded list packing) against plain numpy restatements, including the reference's error
behaviour (trie.py:128-131: ids outside int32, lengths that do not line up)."""

import numpy as np
import pytest

from paper_2508_11553_b200 import SpanOrigin
from paper_2508_11553_b200.trie import runs_from_per_token

_tmfast = pytest.importorskip("paper_2508_11553_b200._tmfast")
OUT, IN = SpanOrigin.MODEL_OUTPUT, SpanOrigin.AGENT_INPUT


def _meta(origins, versions):
    st, org, ver, k = _tmfast.meta_runs(origins, versions, OUT, IN)
    return np.frombuffer(st, np.int32, k), np.frombuffer(org, np.uint8, k), np.frombuffer(ver, np.int32, k)


def test_meta_runs_matches_restatement_random():
    rng = np.random.default_rng(11)
    for trial in range(900):
        n = int(rng.integers(1, 400))
        o = rng.integers(0, 2, n)
        if rng.random() < 0.5:  # long runs (the identity scan) or per-token noise
            o = np.resize(np.repeat(o[: max(1, n // 20)], 20), n)
        step = 0.5 if trial % 2 else 0.05
        v = np.cumsum(rng.random(n) < step).astype(np.int64) * (1 if rng.random() < 0.5 else 1_000_003)
        kind = trial % 3  # this package's enum, bools, 0/1 ints
        origins = [OUT if x else IN for x in o] if kind == 0 else [bool(x) for x in o] if kind == 1 else o.tolist()
        got = _meta(origins, v.tolist())
        want = runs_from_per_token(o.astype(np.int64), v)
        for g, w in zip(got, want):
            assert np.array_equal(np.asarray(g, np.int64), np.asarray(w, np.int64)), trial


def test_meta_runs_many_runs_and_errors():
    n = 5000  # more runs than the extension's inline buffer: the heap path
    o = [OUT if i % 2 else IN for i in range(n)]
    st, org, ver = _meta(o, [0] * n)
    assert len(st) == n and st.tolist() == list(range(n)) and org.tolist() == [i % 2 for i in range(n)]
    with pytest.raises(ValueError):
        _tmfast.meta_runs([IN, IN], [0], OUT, IN)  # not parallel
    with pytest.raises((ValueError, OverflowError)):
        _tmfast.meta_runs([IN] * 3, [0, 2**40, 1], OUT, IN)  # version outside int32
    assert _tmfast.meta_runs([], [], OUT, IN)[3] == 0


def test_pack_i32_and_pack_lists():
    rng = np.random.default_rng(12)
    toks = rng.integers(-(2**31), 2**31 - 1, 10_000).tolist()
    assert np.array_equal(np.frombuffer(_tmfast.pack_i32(toks), np.int32), np.asarray(toks, np.int32))
    assert np.array_equal(np.frombuffer(_tmfast.pack_i32(tuple(toks[:7])), np.int32), np.asarray(toks[:7], np.int32))
    big = [1, 2**31, 3]  # the reference's ValueError for ids outside int32
    with pytest.raises(ValueError):
        _tmfast.pack_i32(big)
    rows = [rng.integers(0, 151_936, int(rng.integers(0, 3000))).tolist() for _ in range(200)]
    for nthreads in (1, 4):
        tok, off = _tmfast.pack_lists(rows, nthreads)
        tok, off = np.frombuffer(tok, np.int32), np.frombuffer(off, np.int64)
        assert off[0] == 0 and np.array_equal(np.diff(off), [len(r) for r in rows])
        assert np.array_equal(tok, np.concatenate([np.asarray(r, np.int32) for r in rows]))
    with pytest.raises(ValueError):
        _tmfast.pack_lists([[1, 2], [2**40]], 2)


def test_meta_runs_fast_path_equals_python_path(monkeypatch):
    """trie.meta_runs with the extension and with its pure-Python path (lists, tuples,
    numpy integer versions, this package's enum and bools) give the same runs."""
    from paper_2508_11553_b200 import trie as T

    rng = np.random.default_rng(13)
    for trial in range(600):
        n = int(rng.integers(1, 200))
        o = rng.integers(0, 2, n)
        if rng.random() < 0.6:
            o = np.resize(np.repeat(o[: max(1, n // 10)], 10), n)
        v = np.cumsum(rng.random(n) < 0.1).astype(np.int64)
        origins = [OUT if x else IN for x in o] if trial % 2 else [bool(x) for x in o]
        versions = [int(x) for x in v] if trial % 3 else [np.int64(x) for x in v]
        if trial % 4 == 1:
            origins, versions = tuple(origins), tuple(versions)
        fast = T.meta_runs(origins, versions)
        monkeypatch.setattr(T, "_tmfast", None)
        slow = T.meta_runs(origins, versions)
        monkeypatch.setattr(T, "_tmfast", _tmfast)
        for f, s in zip(fast, slow):
            assert np.array_equal(np.asarray(f, np.int64), np.asarray(s, np.int64)), trial
