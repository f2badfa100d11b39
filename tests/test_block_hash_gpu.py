"""tm_block_hashes (the per-block hash of the north star's hash-first filter, kept for the
A/B in bench.py) against a numpy restatement of the same mixing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

def fmix32(h):
    h = h.astype(np.uint32)
    with np.errstate(over="ignore"):
        h = h ^ (h >> np.uint32(16))
        h = h * np.uint32(0x85EBCA6B)
        h = h ^ (h >> np.uint32(13))
        h = h * np.uint32(0xC2B2AE35)
        h = h ^ (h >> np.uint32(16))
    return h


def block_hash_ref(tok):
    w = tok.view(np.uint32).reshape(-1, 32, 4)
    k = (np.uint32(2) * np.arange(32, dtype=np.uint32) + np.uint32(1))[None, :]
    with np.errstate(over="ignore"):
        a = fmix32((w[:, :, 0] * np.uint32(0x9E3779B1) + w[:, :, 1] * np.uint32(0x85EBCA77)) ^ (k * np.uint32(0x27D4EB2F)))
        c = fmix32((w[:, :, 2] * np.uint32(0xC2B2AE3D) + w[:, :, 3] * np.uint32(0x165667B1)) ^ (k * np.uint32(0x9E3779B1)))
        a = np.bitwise_xor.reduce(a, axis=1)
        c = np.bitwise_xor.reduce(c, axis=1)
        hi = fmix32(a ^ np.uint32(0x5BD1E995)).astype(np.uint64)
        lo = fmix32(c + a).astype(np.uint64)
    return (hi << np.uint64(32)) | lo


def test_block_hashes_match_restatement():
    import torch

    from paper_2508_11553_b200 import DeviceStore

    rng = np.random.default_rng(4)
    tok = rng.integers(-(2**31), 2**31 - 1, 128 * 1000, dtype=np.int64).astype(np.int32)
    tok[128:256] = tok[:128]  # equal blocks hash equal
    st = DeviceStore(0)
    try:
        dt = torch.from_numpy(tok).cuda()
        out = torch.empty(1000, dtype=torch.int64, device="cuda")
        st.block_hashes(dt, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, block_hash_ref(tok))
        assert got[0] == got[1] and len(set(got.tolist())) == 999
        with pytest.raises(ValueError):
            st.block_hashes(dt[:100], out)
    finally:
        st.close()
