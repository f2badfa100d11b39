"""Routed (cross-GPU, fused P2P) match: world size 1 in-process and world size 2 under
torchrun when two GPUs are visible."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29561", os.path.join(ROOT, "tests", "mp", "routed_match.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "ROUTED_OK=1" in out.stdout, out.stdout[-3000:]


def test_routed_match_world1():
    _run(1)


def test_routed_match_world2():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    _run(2)


def test_device_barrier_peer_timeout_is_a_loud_error():
    """A peer that never arrives at the device-side barrier becomes a device error after
    TM_PEER_TIMEOUT_MS (here 300 ms) instead of hanging the stream."""
    env = dict(os.environ, TM_PEER_TIMEOUT_MS="300")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "mp", "peer_timeout.py")], env=env,
                         capture_output=True, text=True, timeout=120)
    assert "DEVICE_ERROR" in out.stdout and "peer rank timed out" in out.stdout, out.stdout + out.stderr
