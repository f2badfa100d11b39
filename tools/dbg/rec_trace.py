import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2508_11553_b200 import DeviceStore
from workloads import RecordWorkload
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = RecordWorkload(cfg)
sids, tok, off, roff, rs, ro, rv = wl.packed()
lens = np.diff(off)
pad = (lens + 31) // 32 * 32
aoff = np.zeros(len(lens) + 1, np.int64); np.cumsum(pad, out=aoff[1:])
atok = np.zeros(int(aoff[-1]), np.int32)
for k in range(len(lens)):
    atok[aoff[k]: aoff[k] + lens[k]] = tok[off[k]: off[k + 1]]
dtok = torch.from_numpy(atok).cuda()
store = DeviceStore(0, arena_words=6 * int(aoff[-1]) + (1 << 22), row_capacity=6 * len(lens) + 64,
                    run_capacity=6 * len(rs) + 64, session_capacity=6 * wl.n_sessions + 16)
for rep in range(4):
    smap = [store.new_session() for _ in range(wl.n_sessions)]
    g = np.asarray([smap[s] for s in sids], np.int32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = store.record_device(g, dtok, aoff[:-1], lens, roff, rs, ro, rv)
    t1 = time.perf_counter()
    print(f"record_device call {1e3*(t1-t0):.3f} ms", file=sys.stderr)
