"""tm_block_hashes (the per-block hash of the north star's hash-first filter, kept for the
A/B in bench.py) against a numpy restatement of the same mixing."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

M = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(x):
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def block_hash_ref(tok):
    w = tok.astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    w = w.reshape(-1, 32, 4)
    lane = np.arange(32, dtype=np.uint64)
    g = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        a = mix64(((w[:, :, 0] << np.uint64(32)) | w[:, :, 1]) + g * (np.uint64(2) * lane + np.uint64(1)))
        b = mix64(((w[:, :, 2] << np.uint64(32)) | w[:, :, 3]) + g * (np.uint64(2) * lane + np.uint64(2)))
    h = np.bitwise_xor.reduce(a ^ b, axis=1)
    return mix64(h)


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
