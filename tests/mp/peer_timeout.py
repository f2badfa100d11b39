"""Subprocess for tests/test_routing_gpu.py: a routed match with device-side barriers where
one peer never arrives must end as a loud device error after TM_PEER_TIMEOUT_MS, not hang."""

import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

from paper_2508_11553_b200 import DeviceStore  # noqa: E402
from paper_2508_11553_b200._lib import check  # noqa: E402
from paper_2508_11553_b200.routing import route_layout  # noqa: E402

store = DeviceStore(0)
off, nbytes = route_layout(4, 1024)
regions = []
for _ in range(2):  # this rank's region and a "peer" region nobody ever signals into
    ptr = C.c_void_p()
    check(store.lib.tm_shared_alloc(store.h, nbytes, C.byref(ptr)))
    regions.append(ptr.value)
peers = (C.c_void_p * 2)(*regions)
g2l = torch.full((4,), -1, dtype=torch.int32, device="cuda")
check(store.lib.tm_route_prepare(store.h, C.c_void_p(regions[0]), 0, (C.c_int64 * 12)(*off), 2, 0, None))
check(store.lib.tm_match_routed_sync(store.h, 2, 0, peers, C.c_void_p(g2l.data_ptr()), g2l.numel(), 1, None))
t0 = time.time()
try:
    store.synchronize()
    print("NO_ERROR")
except RuntimeError as e:
    print(f"DEVICE_ERROR after {time.time() - t0:.2f}s: {e}")
