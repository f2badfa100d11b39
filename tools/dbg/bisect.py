import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_11553_b200 import DeviceStore
mode = sys.argv[2] if len(sys.argv) > 2 else "last"
for k in [int(x) for x in sys.argv[1].split(",")]:
    store = DeviceStore(0)
    sid = store.new_session()
    L = 1 << k
    rng = np.random.default_rng(k)
    h = rng.integers(-(2**31), 2**31 - 1, L, dtype=np.int64).astype(np.int32) if "neg" in mode else rng.integers(0, 1000, L).astype(np.int32)
    one = (np.array([0], np.int32), np.array([1], np.uint8), np.array([0], np.int32))
    r = store.record([sid], [h], [one])
    b = h.copy()
    pos = L - 1 if "last" in mode else L // 2
    b[pos] ^= 1
    try:
        r = store.record([sid], [b], [one])
        print(k, "ok", r.matched, flush=True)
    except Exception as e:
        print(k, "FAIL", str(e)[:80], flush=True)
        break
    store.close()
