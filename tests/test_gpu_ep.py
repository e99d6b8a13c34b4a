"""Expert-parallel layer on real GPUs over NCCL (needs >= 2 GPUs): launches
tests/ep_gpu_check.py under torchrun and requires bit-identical routing and
outputs against the single-GPU layer."""

import os
import subprocess
import sys

import pytest
import torch

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def test_ep_matches_single_gpu():
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "tests", "ep_gpu_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-5000:]
    assert res.stdout.count("transport=nccl") == 5
    assert res.stdout.count("transport=p2p ") == 2
    assert res.stdout.count("transport=p2p-chunked") == 4
    if n % 2 == 0:
        assert res.stdout.count("schedule=hierarchical") == 3
    assert res.stdout.count("schedule=coordinated") >= 3
    assert res.stdout.count("random-case") >= 4
