"""torchrun worker for tests/test_routing_gpu.py: c5-style routed match across ranks,
checked against the constructed truth and against the owner's host-path match."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_2508_11553_b200 import DeviceStore  # noqa: E402
from paper_2508_11553_b200.routing import Router  # noqa: E402
from workloads import C5Workload  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
wl = C5Workload(3000, lo=64, hi=20000, nranks=world, rank=rank, n_queries=700)
store = DeviceStore(local)
wl.build_shard(store)
need = torch.tensor([int(wl.q_off[-1])], device=dev)
dist.all_reduce(need, op=dist.ReduceOp.MAX)
router = Router(store, dist.group.WORLD, n_max=wl.n_queries, tokens_max=int(need.item()), g2l=wl.g2l)
wl.fill_queries(router)
for _ in range(3):
    router.match(wl.n_queries)  # device-side barriers (default)
torch.cuda.synchronize()
store.synchronize()  # raises if a peer timed out
m = router.out_matched[: wl.n_queries].cpu().numpy()
par = router.out_parent[: wl.n_queries].cpu().numpy()
ok = np.array_equal(m, wl.q_depth) and bool(np.all((par >= 0) | (m == 0)))
# the fused path with NCCL barriers, and the NCCL-only baseline exchange, must agree exactly
for sync in ("nccl", "device"):
    router.out_matched.fill_(-7)
    router.match(wl.n_queries, sync=sync)
    torch.cuda.synchronize()
    ok = ok and np.array_equal(router.out_matched[: wl.n_queries].cpu().numpy(), m)
# an id beyond 18 bits (past every query's compared prefix: results unchanged) makes this
# rank's owners read the int32 tokens instead of the packed planes
i0 = int(np.argmax(wl.q_len - wl.q_depth > 8))
pos = int(wl.q_off[i0] + wl.q_depth[i0] + 5)
saved = int(router.tokens[pos].item())
router.tokens[pos] = 1 << 20
router.out_matched.fill_(-7)
router.match(wl.n_queries)
torch.cuda.synchronize()
ok = ok and np.array_equal(router.out_matched[: wl.n_queries].cpu().numpy(), m)
ok = ok and np.array_equal(router.out_parent[: wl.n_queries].cpu().numpy(), par)
router.tokens[pos] = saved
router.out_matched.fill_(-7)
router.match_nccl(wl.n_queries)
torch.cuda.synchronize()
ok = ok and np.array_equal(router.out_matched[: wl.n_queries].cpu().numpy(), m)
ok = ok and np.array_equal(router.out_parent[: wl.n_queries].cpu().numpy(), par)
# ragged edge cases: empty, one-token, sub-group and group-straddling queries (the pack skips
# empty queries and zero-fills partial 32-position groups); truth = min(length, depth)
short = np.array(wl.q_len, np.int64)
sel = np.arange(0, wl.n_queries, 7)
short[sel] = np.resize(np.array([0, 1, 5, 31, 33, 4097], np.int64), len(sel))
short = np.minimum(short, wl.q_len)
router.qlen[: wl.n_queries].copy_(torch.as_tensor(short, device=dev))
for sync in ("device", "nccl"):
    router.out_matched.fill_(-7)
    router.match(wl.n_queries, sync=sync)
    torch.cuda.synchronize()
    ok = ok and np.array_equal(router.out_matched[: wl.n_queries].cpu().numpy(), np.minimum(short, wl.q_depth))
router.qlen[: wl.n_queries].copy_(torch.as_tensor(wl.q_len, device=dev))
# pipelined: two regions, batch i+1 bucketed + packed on a side stream while batch i matches
from paper_2508_11553_b200.routing import match_pipelined  # noqa: E402

router2 = Router(store, dist.group.WORLD, n_max=wl.n_queries, tokens_max=int(need.item()), g2l=wl.g2l)
wl.fill_queries(router2)
for r in (router, router2):
    r.out_matched.fill_(-7)
torch.cuda.synchronize()
match_pipelined([router, router2], wl.n_queries, 5)
torch.cuda.synchronize()
store.synchronize()
for r in (router, router2):
    ok = ok and np.array_equal(r.out_matched[: wl.n_queries].cpu().numpy(), m)
    ok = ok and np.array_equal(r.out_parent[: wl.n_queries].cpu().numpy(), par)
router2.close()
# push routing: requesters write the remote queries' planes into the owners' inboxes
# (one batch, the big-id fallback, ragged lengths, and pipelined over two regions)
if world > 1:
    pr = [Router(store, dist.group.WORLD, n_max=wl.n_queries, tokens_max=int(need.item()), g2l=wl.g2l, push=True)
          for _ in range(2)]
    for r in pr:
        wl.fill_queries(r)
        r.out_matched.fill_(-7)
    pr[0].match(wl.n_queries)
    torch.cuda.synchronize()
    ok = ok and np.array_equal(pr[0].out_matched[: wl.n_queries].cpu().numpy(), m)
    ok = ok and np.array_equal(pr[0].out_parent[: wl.n_queries].cpu().numpy(), par)
    ok = ok and np.array_equal(pr[0].out_dup[: wl.n_queries].cpu().numpy(), router.out_dup[: wl.n_queries].cpu().numpy())
    pr[0].tokens[pos] = 1 << 20
    pr[0].out_matched.fill_(-7)
    pr[0].match(wl.n_queries)
    torch.cuda.synchronize()
    ok = ok and np.array_equal(pr[0].out_matched[: wl.n_queries].cpu().numpy(), m)
    pr[0].tokens[pos] = saved
    pr[0].qlen[: wl.n_queries].copy_(torch.as_tensor(short, device=dev))
    pr[0].out_matched.fill_(-7)
    pr[0].match(wl.n_queries)
    torch.cuda.synchronize()
    ok = ok and np.array_equal(pr[0].out_matched[: wl.n_queries].cpu().numpy(), np.minimum(short, wl.q_depth))
    pr[0].qlen[: wl.n_queries].copy_(torch.as_tensor(wl.q_len, device=dev))
    for r in pr:
        r.out_matched.fill_(-7)
    torch.cuda.synchronize()
    match_pipelined(pr, wl.n_queries, 5)
    torch.cuda.synchronize()
    store.synchronize()
    for r in pr:
        ok = ok and np.array_equal(r.out_matched[: wl.n_queries].cpu().numpy(), m)
        ok = ok and np.array_equal(r.out_parent[: wl.n_queries].cpu().numpy(), par)
    print(f"rank {rank} push ok={ok}", flush=True)
    for r in pr:
        r.close()
remote = float(np.mean(wl.owner[wl.q_g] != rank))
flag = torch.tensor([1 if ok else 0], device=dev)
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print(f"ROUTED_OK={int(flag.item())} world={world} remote_frac={remote:.2f}")
router.close()
store.close()
dist.destroy_process_group()
