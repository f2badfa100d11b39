"""Host-side routing logic (CPU, gloo world_size 2): owner hashing agrees with an
independent restatement, every session has exactly one owner, and the routing
region layout keeps arrays disjoint and aligned."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2508_11553_b200.routing import owner_of, route_layout


def _splitmix_owner(g, n):
    x = (g + 0x9E3779B97F4A7C15) & (2**64 - 1)
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & (2**64 - 1)
    x ^= x >> 31
    return x % n


def test_owner_of_matches_restatement():
    ids = list(range(0, 5000)) + [2**40 + 7, 123456789012]
    for n in (1, 2, 3, 8):
        got = owner_of(ids, n)
        assert [int(x) for x in got] == [_splitmix_owner(g, n) for g in ids]
    counts = np.bincount(owner_of(np.arange(200_000), 8), minlength=8)
    assert counts.min() > 0.97 * 25_000 and counts.max() < 1.03 * 25_000


def test_route_layout_disjoint_and_aligned():
    off, total = route_layout(4096, 1_000_000, header=16_000)
    assert off[0] >= 16_000
    planes = (1_000_000 + 63) // 64 * 64 + 128  # 18-bit planes with 64-position copy granules of slack
    sizes = [8 * 4096, 8 * 4096, 8 * 4096, 4 * 1_000_000, 4 * 4096, 8 * 4096, 8 * 4096, 8 * 4096, 2 * planes,
             planes // 4, 4 * 4097, 32 * 4096]
    assert len(off) == 12
    for (a, s), b in zip(zip(off, sizes), off[1:] + [total]):
        assert a % 256 == 0 and a + s <= b


def test_route_layout_push_inbox_slices():
    """Push routing: nranks slices of (low plane, high plane, records) at one stride, past
    every other array, so slice p of one rank's region is written only by rank p."""
    n, t, r = 4096, 1_000_000, 4
    off, total, stride = route_layout(n, t, header=16_000, inbox=r)
    planes = (t + 63) // 64 * 64 + 128
    lo, hi, pk, rec = off[8:]
    assert lo % 256 == 0 and hi % 256 == 0 and rec % 256 == 0 and stride % 256 == 0
    assert lo + 2 * planes <= hi and hi + planes // 4 <= rec and rec + 32 * n <= lo + stride
    assert pk + 4 * (n + 1) <= lo and max(off[:8]) < pk
    assert total == lo + r * stride
    flat, _ = route_layout(n, t, header=16_000)
    assert off[:8] == flat[:8]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from workloads import C5Workload

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    wl = C5Workload(20_000, nranks=world, rank=rank, n_queries=256)
    owned = [None] * world
    dist.all_gather_object(owned, wl.owned.tolist())
    # every requester computes the same owner for each of its queries as the owners do
    mine = set(wl.owned.tolist())
    q.put((rank, len(mine), sorted(set().union(*map(set, owned))) == list(range(20_000)),
           sum(len(o) for o in owned), int(wl.q_off[-1]), bool(np.all(wl.g2l[wl.owned] == np.arange(len(wl.owned))))))
    dist.destroy_process_group()


def test_sharding_partitions_sessions_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in ps]
    res = sorted(q.get(timeout=120) for _ in ps)
    [p.join(timeout=60) for p in ps]
    assert all(p.exitcode == 0 for p in ps)
    assert res[0][2] and res[1][2]                 # union of owned sets = all sessions
    assert res[0][3] == 20_000                     # ... and they are disjoint
    assert res[0][1] + res[1][1] == 20_000
    assert res[0][5] and res[1][5]
