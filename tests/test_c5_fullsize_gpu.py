"""Config 5 at full size on one GPU: the 1M-session store (log-uniform 1k-128k histories,
~107 GB) and a 4,096-query batch routed through Router.match, checked on every query
against the constructed depth and on a sample of 512 queries against the C restatement of
the reference trie, with the sampled sessions' histories and queries regenerated on the
CPU from the same counter-based generator (matched length, parent row, duplicate row)."""

import numpy as np
import pytest

from oracle.cport import CRadixStore

pytestmark = pytest.mark.gpu


def test_c5_one_gpu_vs_oracle_sample():
    import torch
    import torch.distributed as dist

    from paper_2508_11553_b200 import DeviceStore
    from paper_2508_11553_b200.routing import Router
    from workloads import VOCAB, C5Workload, synth_tokens, turn_runs_batch

    own_pg = not dist.is_initialized()
    if own_pg:
        dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29577", rank=0, world_size=1)
    wl = C5Workload(1_000_000, nranks=1, rank=0, n_queries=4096)
    owned_tokens = int(((wl.lens + 31) // 32 * 32).sum())
    store = DeviceStore(0, arena_words=owned_tokens + (1 << 22), row_capacity=len(wl.owned) + 64,
                        run_capacity=16 * len(wl.owned) + 64, session_capacity=len(wl.owned) + 16)
    try:
        wl.build_shard(store)
        router = Router(store, dist.group.WORLD, n_max=wl.n_queries, tokens_max=int(wl.q_off[-1]), g2l=wl.g2l)
        wl.fill_queries(router)
        router.match(wl.n_queries)
        torch.cuda.synchronize()
        m = router.out_matched[: wl.n_queries].cpu().numpy()
        par = router.out_parent[: wl.n_queries].cpu().numpy()
        dup = router.out_dup[: wl.n_queries].cpu().numpy()
        assert np.array_equal(m, wl.q_depth)
        # the sample: histories and queries regenerated on the CPU
        rng = np.random.default_rng(3)
        pick = np.sort(rng.choice(wl.n_queries, 512, replace=False))
        sess = np.unique(wl.q_g[pick])
        local = {int(g): k for k, g in enumerate(sess)}
        lens = wl.lens[sess]
        hoff = np.r_[0, np.cumsum(lens)]
        g_t = torch.repeat_interleave(torch.as_tensor(sess), torch.as_tensor(lens))
        pos = torch.arange(int(hoff[-1]), dtype=torch.int64) - torch.repeat_interleave(torch.as_tensor(hoff[:-1]),
                                                                                      torch.as_tensor(lens))
        hist = synth_tokens(g_t, pos).numpy()
        roff, rs, ro, rv = turn_runs_batch(lens)
        ora = CRadixStore()
        ora.insert_batch(np.arange(len(sess), dtype=np.int32), hist, hoff, roff, rs, ro, rv, nthreads=8)
        qt, qo = [], [0]
        for i in pick:
            g, d, L = int(wl.q_g[i]), int(wl.q_depth[i]), int(wl.q_len[i])
            p = torch.arange(L, dtype=torch.int64)
            gi = torch.full((L,), g, dtype=torch.int64)
            h = synth_tokens(gi, p)
            fresh = synth_tokens(gi, p, salt=1)
            forced = ((h.to(torch.int64) + 1 + synth_tokens(gi, p, salt=2).to(torch.int64) % (VOCAB - 1)) % VOCAB).to(torch.int32)
            Lh = int(wl.lens[g])
            q = torch.where(p < d, h, torch.where((p == d) & (d < Lh), forced, fresh)).numpy()
            qt.append(q)
            qo.append(qo[-1] + L)
        mo, po, do = ora.match_batch(np.asarray([local[int(g)] for g in wl.q_g[pick]], np.int32), np.concatenate(qt),
                                     np.asarray(qo, np.int64), nthreads=8)
        assert np.array_equal(m[pick], mo)
        # one row per session: parent / dup as session-local ordinals
        loc = lambda rows: np.array([store.row_info(int(x))["local"] if x >= 0 else -1 for x in rows])  # noqa: E731
        assert np.array_equal(loc(par[pick]), po)
        assert np.array_equal(loc(dup[pick]), do)
        router.close()
    finally:
        store.close()
        if own_pg:
            dist.destroy_process_group()
