import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_11553_b200 import DeviceStore, SessionTrie, SpanOrigin
store = DeviceStore(0)
trie = SessionTrie("x", store=store)
rng = np.random.default_rng(0)
base = rng.integers(0, 151936, 16).tolist()
org = [SpanOrigin.AGENT_INPUT] * 8 + [SpanOrigin.MODEL_OUTPUT] * 8
for i in range(30):
    s = base[:8] + rng.integers(0, 151936, 8).tolist()
    t0 = time.perf_counter(); trie.lpm_insert(s, org, [0]*16, "c"); print(f"py {1e6*(time.perf_counter()-t0):.1f}", file=sys.stderr)
import torch
x = torch.zeros(1, device="cuda")
for i in range(5):
    t0 = time.perf_counter(); x += 1; torch.cuda.synchronize(); print(f"torch op+sync {1e6*(time.perf_counter()-t0):.1f}", file=sys.stderr)
