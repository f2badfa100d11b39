import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_11553_b200 import DeviceStore, SessionTrie, SpanOrigin
store = DeviceStore(0)
rng = np.random.default_rng(5)
which = sys.argv[1]
if which == "long":
    trie = SessionTrie("long", store=store)
    L = 1 << 20
    h = rng.integers(-(2**31), 2**31 - 1, L, dtype=np.int64).astype(np.int32)
    ins = lambda toks, c: trie.lpm_insert(toks, [SpanOrigin.MODEL_OUTPUT] * len(toks), [7] * len(toks), c)
    print(ins(h, "a"), flush=True)
    b = h.copy(); b[-1] ^= 1
    print(ins(b, "b"), flush=True)
    print(ins(h[: L // 2], "c"), flush=True)
else:
    sid = store.new_session()
    seq = rng.integers(0, 100, 300).tolist()
    n = int(sys.argv[2])
    res = store.record([sid] * n, [seq] * n, [(np.array([0]), np.array([1], np.uint8), np.array([0]))] * n)
    print(res.local[:5], res.added[:5], store.session_stats(sid))
