"""Config 4 / config 5-shard shaped parity (read-only K1 match at full history lengths):
sessions with 32,768-token histories (c4) or log-uniform 1k-128k histories (the c5 shard
slice), some sessions branched by a recorded batch first, then a match batch of 75 %
extensions + 25 % branches with a forced mismatch, through the host-buffer C-ABI call and
the device-tensor call.  Checked against the C restatement of the reference trie
(oracle/radix_oracle.c: matched length, parent row, duplicate row) and against the
constructed depths.  Sizes are scaled down from BASELINE.json's configs so the oracle
finishes in seconds; the bench asserts the same properties at full size."""

import numpy as np
import pytest

from oracle.cport import CRadixStore
from workloads import MatchWorkload

pytestmark = pytest.mark.gpu


def _local(store, rows):
    return np.array([store.row_info(int(x))["local"] if x >= 0 else -1 for x in rows])


@pytest.mark.parametrize("shape", ["c4", "c5-shard"])
def test_match_batch_vs_c_oracle(shape):
    import torch

    from paper_2508_11553_b200 import DeviceStore

    if shape == "c4":
        wl = MatchWorkload(160, 32_768, 768, seed=91)
    else:
        wl = MatchWorkload(96, n_queries=384, mixed=(1024, 131_072), seed=92)
    ns = wl.n_sessions
    ora = CRadixStore()
    toks = np.concatenate([wl.hist_tokens[wl.hist_off[s]: wl.hist_off[s] + wl.hist_len[s]] for s in range(ns)])
    off = np.zeros(ns + 1, np.int64)
    np.cumsum(wl.hist_len, out=off[1:])
    ora.insert_batch(np.arange(ns, dtype=np.int32), toks, off, wl.run_off, wl.run_start, wl.run_origin,
                     wl.run_version, nthreads=4)
    store = DeviceStore(0)
    try:
        sids = [store.new_session() for _ in range(ns)]
        assert sids == list(range(ns))
        store.record_packed(np.arange(ns, dtype=np.int32), wl.hist_tokens, wl.hist_off[:-1].copy(), wl.hist_len,
                            wl.run_off, wl.run_start, wl.run_origin, wl.run_version)

        def flat(q, k=None):
            idx = range(len(q["q_sess"])) if k is None else k
            t = [q["q_tokens"][q["q_off"][i]: q["q_off"][i] + q["q_len"][i]] for i in idx]
            o = np.zeros(len(t) + 1, np.int64)
            np.cumsum([len(x) for x in t], out=o[1:])
            return np.concatenate(t), o

        # branch some sessions first: record a third of a first batch (new rows off the
        # history at the branch depth, or extensions of it) into both stores
        first = wl.make_queries(np.random.default_rng(7))
        pick = np.arange(0, len(first["q_sess"]), 3)
        ft, fo = flat(first, pick)
        fs = first["q_sess"][pick]
        nrun = len(pick)
        one = np.arange(nrun + 1, dtype=np.int64)
        zs, zo, zv = np.zeros(nrun, np.int32), np.ones(nrun, np.uint8), np.ones(nrun, np.int32)
        om, orow, opar, oadd = ora.insert_batch(fs, ft, fo, one, zs, zo, zv, nthreads=4)
        r = store.record_packed(fs, ft, fo[:-1].copy(), np.diff(fo), one, zs, zo, zv)
        assert np.array_equal(r.matched, om) and np.array_equal(r.local, orow)
        assert np.array_equal(r.parent_local, opar) and np.array_equal(r.added, oadd)

        # the match batch: the workload's own queries plus, off the branch rows recorded
        # above, extensions (parent = that row), exact copies (dup = that row) and strict
        # prefixes; 32-aligned starts like the workload's layout
        q = wl.make_queries(np.random.default_rng(8))
        rng = np.random.default_rng(9)
        extra_s, extra_t = [], []
        for k in range(0, nrun, 2):
            row = ft[fo[k]: fo[k + 1]]
            extra_s += [fs[k]] * 3
            extra_t += [np.concatenate([row, rng.integers(0, 151936, 100, dtype=np.int32)]), row, row[: len(row) - 7]]
        lens = np.concatenate([q["q_len"], [len(x) for x in extra_t]]).astype(np.int64)
        qoff = np.zeros(len(lens) + 1, np.int64)
        np.cumsum((lens + 31) // 32 * 32, out=qoff[1:])
        qtok = np.zeros(int(qoff[-1]), np.int32)
        for i, x in enumerate([q["q_tokens"][q["q_off"][i]: q["q_off"][i] + q["q_len"][i]]
                               for i in range(len(q["q_sess"]))] + extra_t):
            qtok[qoff[i]: qoff[i] + len(x)] = x
        nq0 = len(q["q_sess"])
        q = dict(q_sess=np.concatenate([q["q_sess"], np.array(extra_s, np.int32)]), q_len=lens, q_off=qoff,
                 q_tokens=qtok, q_depth=np.concatenate([q["q_depth"], lens[nq0:]]))
        qt, qo = flat(q)
        m_o, p_o, d_o = ora.match_batch(q["q_sess"], qt, qo, nthreads=4)
        # positions before the forced mismatch are history: the constructed depth bounds
        # the match from below (a branch recorded above can only extend it)
        assert np.all(m_o[:nq0] >= np.minimum(q["q_depth"][:nq0], q["q_len"][:nq0]))
        assert np.all(m_o[nq0:] >= lens[nq0:] - 100) and np.any(p_o > 0) and np.any(d_o >= 0)
        m_h, p_h, d_h = store.match(q["q_sess"], q["q_tokens"], q["q_off"][:-1].copy(), q["q_len"])
        assert np.array_equal(m_h, m_o)
        assert np.array_equal(_local(store, p_h), p_o)
        assert np.array_equal(_local(store, d_h), d_o)
        dev = torch.device("cuda", 0)
        t = [torch.from_numpy(np.ascontiguousarray(x)).to(dev)
             for x in (q["q_sess"], q["q_tokens"], q["q_off"][:-1], q["q_len"])]
        outs = [torch.empty(len(q["q_sess"]), dtype=torch.int64, device=dev) for _ in range(3)]
        store.match_device(*t, *outs)
        torch.cuda.synchronize()
        assert np.array_equal(outs[0].cpu().numpy(), m_o)
        assert np.array_equal(outs[1].cpu().numpy(), p_h)
        assert np.array_equal(outs[2].cpu().numpy(), d_h)
    finally:
        store.close()
