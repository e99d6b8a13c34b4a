"""Randomised parity sweep of the bf16 layer (seeded): shapes, k, capacity
factor, residual / fused / unfused paths drawn at random, each checked against
the oracle on the device's own logits (routing bit-exact, outputs to the bf16
tolerance of test_gpu_layer). Exercises the GEMM variants (1-/2-CTA, BN
32..256, TMA-store epilogue, dynamic tile scheduler) across ragged group sizes."""

import os

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2201_05596_b200 import arch as A
from paper_2201_05596_b200.gating import GatingConfig
from tests.test_gpu_layer import check_routing, close, oracle_args, rounded_params, run_layer

pytestmark = pytest.mark.gpu


# MOE_STRESS_N / MOE_STRESS_SEED: a longer sweep with other seeds (the default suite
# runs the first 40 / 10 cases of seed 0)
_N = int(os.environ.get("MOE_STRESS_N", "40"))
_SEED = int(os.environ.get("MOE_STRESS_SEED", "0"))


def _draw(i):
    r = np.random.default_rng(1000 + i + 100003 * _SEED)
    M = int(r.choice([64, 128, 256, 512]))
    E = int(r.integers(1, 65))
    k = 1 if E == 1 else int(r.choice([1, 2]))
    S = int(r.integers(1, 3000))
    cf = float(r.uniform(0.3, 2.0))
    res = bool(r.random() < 0.3)
    fuse = bool(r.random() < 0.7)
    return S, M, E, k, cf, res, fuse


@pytest.mark.parametrize("i", range(_N))
def test_random_layer(i):
    S, M, E, k, cf, res, fuse = _draw(i)
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=res, gating=GatingConfig(E, k, cf))
    p = rounded_params(spec, 77 + i, torch.bfloat16)
    x64 = torch.randn(S, M, generator=torch.Generator().manual_seed(i)).to(torch.bfloat16)
    x64 = x64.double().numpy()
    layer, x, out, logits = run_layer(spec, p, x64, torch.bfloat16, fuse=fuse)
    lg, _ = check_routing(layer, logits, spec, S)
    ex, sh = oracle_args(p)
    want = O.forward_layer_with_logits(x64, lg, ex, sh, E, k, cf)
    close(out.float().cpu().numpy(), want, 2e-2)


@pytest.mark.parametrize("i", range(max(_N // 4, 10)))
def test_random_backward(i):
    """The training path (forward_train + backward) at random shapes against the
    oracle's closed-form backward on the device logits (tolerances of
    test_gpu_train)."""
    from tests.test_gpu_train import test_backward_vs_oracle_on_device_logits as check

    r = np.random.default_rng(5000 + i + 100003 * _SEED)
    M = int(r.choice([64, 128, 256]))
    E = int(r.integers(2, 33))
    k = int(r.choice([1, 2]))
    S = int(r.integers(64, 2500))
    cf = float(r.uniform(0.4, 1.6))
    res = bool(r.random() < 0.4)
    # dx passes through four bf16 roundings (dY, dA, dXr, the gate term's hi/lo) whose
    # intermediates can exceed dx itself: over long sweeps an element in ~10^6 lands
    # at 2-2.1% of (|dx| + RMS) - deterministic and spread over experts
    # (tools/dbg/bwd_case_dbg.py), so the sweep uses the weight-gradient tolerance;
    # the weight gradients (bf16 h and dY, GELU' from the bf16 pre-activation) likewise
    # reach 3.5% on one element in a 200-case sweep (seed 21, case 4: S=501, k=2,
    # Residual-MoE, cap 21; deterministic)
    check(S, M, E, k, cf, res, dx_rtol=3e-2, w_rtol=4e-2)


@pytest.mark.parametrize("i", range(8))
def test_random_layer_odd_width(i):
    """d_model a multiple of 8 but not of 32: the epilogues' partial 32-column
    chunks (scalar tails of the combine / Residual-MoE epilogues, BN 64 / 128 /
    256 tiles with a ragged last block)."""
    r = np.random.default_rng(3000 + i)
    M = int(r.choice([40, 72, 136, 200]))
    E = int(r.integers(2, 20))
    k = int(r.choice([1, 2]))
    S = int(r.integers(300, 2500))
    cf = float(r.uniform(0.5, 2.0))
    res = bool(i % 2)
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=res, gating=GatingConfig(E, k, cf))
    p = rounded_params(spec, 91 + i, torch.bfloat16)
    x64 = torch.randn(S, M, generator=torch.Generator().manual_seed(50 + i)).to(torch.bfloat16)
    x64 = x64.double().numpy()
    layer, x, out, logits = run_layer(spec, p, x64, torch.bfloat16, fuse=bool(i % 3))
    lg, _ = check_routing(layer, logits, spec, S)
    ex, sh = oracle_args(p)
    want = O.forward_layer_with_logits(x64, lg, ex, sh, E, k, cf)
    close(out.float().cpu().numpy(), want, 2e-2)
