"""Time tm_route_prepare (k_route + k_route_pack) on one GPU for a c5-shaped batch with
nranks = 2 (tuning tool): the requester-side cost of packing remote queries."""

import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2508_11553_b200 import DeviceStore  # noqa: E402
from paper_2508_11553_b200._lib import check  # noqa: E402
from paper_2508_11553_b200.routing import _CudaArray, owner_of, route_layout  # noqa: E402


def main(n=4096, nranks=2):
    rng = np.random.default_rng(0)
    lens = np.exp(rng.uniform(np.log(1024), np.log(131072), n)).astype(np.int64)
    pad = (lens + 31) // 32 * 32
    qoff = np.concatenate([[0], np.cumsum(pad)])
    store = DeviceStore(0)
    off, nbytes = route_layout(n, int(qoff[-1]))
    ptr = C.c_void_p()
    check(store.lib.tm_shared_alloc(store.h, nbytes, C.byref(ptr)))
    base = ptr.value
    dev = torch.device("cuda", 0)
    view = lambda i, k, ts: torch.as_tensor(_CudaArray(base + off[i], (k,), ts), device=dev)  # noqa: E731
    gsid = rng.integers(0, 1 << 40, n)
    view(0, n, "<i8").copy_(torch.as_tensor(gsid))
    view(1, n, "<i8").copy_(torch.as_tensor(qoff[:-1]))
    view(2, n, "<i8").copy_(torch.as_tensor(lens))
    view(3, int(qoff[-1]), "<i4").copy_(torch.randint(0, 151936, (int(qoff[-1]),), dtype=torch.int32, device=dev))
    offs = (C.c_int64 * 12)(*off)
    st = torch.cuda.current_stream().cuda_stream
    st = 1 if st == 0 else st  # cudaStreamLegacy: a null handle would mean the store's own stream
    for _ in range(3):
        check(store.lib.tm_route_prepare(store.h, C.c_void_p(base), n, offs, nranks, 0, C.c_void_p(st)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        check(store.lib.tm_route_prepare(store.h, C.c_void_p(base), n, offs, nranks, 0, C.c_void_p(st)))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    tok = int(lens.sum())
    rem = int(lens[owner_of(gsid, nranks) != 0].sum())
    print(f"tm_route_prepare n={n} nranks={nranks} tokens={tok / 1e6:.1f}M (remote {rem / 1e6:.1f}M): "
          f"{ms * 1e3:.1f} us = {6.25 * rem / (ms * 1e-3) / 1e12:.2f} TB/s of pack traffic (4 B read + 2.25 B "
          f"written per remote position) (pack={os.environ.get('TM_ROUTE_PACK', '1')})")


if __name__ == "__main__":
    main()
