import sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, '.')
dev = torch.device('cuda', 0); torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29534", rank=0, world_size=1, device_id=dev)
from paper_2508_11553_b200 import DeviceStore
from paper_2508_11553_b200.routing import Router
from workloads import C5Workload, synth_tokens
wl = C5Workload(2000, n_queries=64)
store = DeviceStore(0)
wl.build_shard(store)
router = Router(store, dist.group.WORLD, n_max=64, tokens_max=int(wl.q_off[-1]), g2l=wl.g2l)
wl.fill_queries(router)
torch.cuda.synchronize()
router.match(64); torch.cuda.synchronize()
m = router.out_matched[:64].cpu().numpy()
print("m", m[:10]); print("d", wl.q_depth[:10]); print("L", wl.lens[wl.q_g][:10])
# host-path match of the same queries
qt = router.tokens[: int(wl.q_off[-1])].cpu().numpy()
sid = wl.g2l[wl.q_g]
mh, ph, dh = store.match(sid, qt, wl.q_off[:-1], wl.q_len)
print("host", mh[:10])
# check stored row vs synth
p = store.export([int(store.session_rows(int(sid[0]))[0])])
g = torch.full((len(p.tokens),), int(wl.q_g[0]), device=dev); pos = torch.arange(len(p.tokens), device=dev)
print("row ok", np.array_equal(p.tokens, synth_tokens(g, pos).cpu().numpy()))
print("q ok", np.array_equal(qt[wl.q_off[0]: wl.q_off[0]+wl.q_depth[0]], synth_tokens(g, pos).cpu().numpy()[:wl.q_depth[0]]))
