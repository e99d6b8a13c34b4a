"""Expert-parallel layer parity on real GPUs: launches tests/ep_gpu_check.py
under torchrun and requires bit-identical routing and outputs against the
single-GPU layer on the concatenated batch.

* ``test_ep_same_device`` runs on ONE B200: two (and four) ranks share cuda:0,
  bootstrapped over gloo; the p2p transport maps the other processes' regions
  with same-device cudaIpc, so ``moe_ipc_allgather_i32``, ``moe_ep_plan``,
  ``moe_dispatch_p2p``, the flag barriers, ``moe_grouped_gemm_bf16_combine_rows``
  and ``moe_pull_rows_p2p`` run exactly as over NVLink; the nccl-transport
  code path runs with its exchanges staged through host memory.
* ``test_ep_matches_single_gpu`` runs one rank per GPU over NCCL/NVLink
  (needs >= 2 GPUs).
"""

import os
import subprocess
import sys

import pytest
import torch

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(n: int, port: int, same_device: bool, timeout: int = 1500) -> str:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "ep_gpu_check.py")]
    env = dict(os.environ, EP_SAME_DEVICE="1" if same_device else "0")
    if same_device:
        env["CUDA_VISIBLE_DEVICES"] = env.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-5000:]
    return res.stdout


def _check_counts(out: str, n: int) -> None:
    assert out.count("transport=nccl") == 5
    assert out.count("transport=p2p ") == 5  # every case: k=2 and Residual-MoE included
    assert out.count("transport=p2p-chunked") == 4
    if n % 2 == 0:
        assert out.count("schedule=hierarchical") == 3
    assert out.count("schedule=coordinated") >= 3
    assert out.count("random-case") >= 4


@pytest.mark.parametrize("n", [2, 4])
def test_ep_same_device(n):
    """EP bit-identity with every rank on one GPU (runs on the 1-GPU box)."""
    out = _run(n, 29541 + n, same_device=True)
    _check_counts(out, n)
    assert out.count("same_device=1") == out.count("ep ok")


if torch.cuda.device_count() >= 2:  # one rank per GPU (collected on multi-GPU boxes only)

    def test_ep_matches_single_gpu():
        n = min(torch.cuda.device_count(), 4)
        out = _run(n, 29533, same_device=False)
        _check_counts(out, n)
