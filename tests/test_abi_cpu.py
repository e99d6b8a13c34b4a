"""CPU-side checks of the boundary: the C ABI library loads, exports every
symbol include/moe_b200.h declares, rejects bad arguments before any launch,
and the Python mirror keeps the reference's config validation."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2201_05596_b200 import _lib
from paper_2201_05596_b200.arch import LayerSpec, ValidationError, init_layer_params
from paper_2201_05596_b200.gating import GatingConfig
from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "moe_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t)\s+(moe_\w+)\s*\(", text, flags=re.M)))


def test_library_builds_and_loads():
    lib = _lib.load()
    assert lib.moe_abi_version() == 1


def test_every_header_symbol_exported_and_bound():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes signature table"
    assert set(_lib.SIGNATURES) == set(syms)


def test_invalid_arguments_rejected_without_launch():
    lib = _lib.load()
    # k = 3, E = 0, bad dtype: all caught before touching the device
    assert lib.moe_topk_gate(None, 0, 4, 8, 3, None, None, None, None) == _lib.MOE_EINVAL
    assert lib.moe_topk_gate(None, 0, 4, 0, 1, None, None, None, None) == _lib.MOE_EINVAL
    assert lib.moe_topk_gate(None, 7, 4, 8, 1, None, None, None, None) == _lib.MOE_EINVAL
    assert lib.moe_blelloch_scan_f64(None, 3, None) == _lib.MOE_EINVAL
    assert lib.moe_gate_gemm_bf16(None, None, 16, 64, 300, 1, None, None, None, None, None,
                                  None) == _lib.MOE_EINVAL
    assert lib.moe_grouped_gemm_bf16(None, 8, 12, None, 8, 8, None, None, 1, None, 0, None, 8,
                                      None, 8, 0, None) == _lib.MOE_EINVAL
    # newer entry points: shape / flag checks come before any device work
    assert lib.moe_grouped_gemm_bf16_wgrad(None, 8, 12, None, 16, 1, 8, None, 8, None,
                                           None) == _lib.MOE_EINVAL          # P % 8
    assert lib.moe_gemm_bf16_wgrad_f32(None, 8, 16, None, 10, None, None) == _lib.MOE_EINVAL
    assert lib.moe_colsum_rows_bf16(None, 12, 1, 0, None, 8, None, None) == _lib.MOE_EINVAL
    assert lib.moe_gather_rows(None, 24, None, 4, None, None) == _lib.MOE_EINVAL  # row_bytes % 16
    assert lib.moe_grouped_gemm_bf16_gather(None, 8, None, 64, None, 64, 64, None, None, 1, 0,
                                            None, 8, 8, 0, None) == _lib.MOE_EINVAL  # row_stride 0
    assert lib.moe_grouped_gemm_bf16(None, 8, 64, None, 8, 8, None, None, 1, None, 0, None, 8,
                                      None, 8, 2 | _lib.MOE_GEMM_PAD_SCRATCH,
                                      None) == _lib.MOE_EINVAL      # act 2 is not a plain GEMM
    assert lib.moe_ep_plan_chunked(None, 4, 0, 6, 1, 8, None, None, None, None, None,
                                   None) == _lib.MOE_EINVAL         # E % world
    assert lib.moe_ep_plan_chunked(None, 2, 0, 8, 0, 8, None, None, None, None, None,
                                   None) == _lib.MOE_EINVAL         # chunks >= 1
    assert lib.moe_set_launch_limits(-1, 0) == _lib.MOE_EINVAL
    assert lib.moe_set_launch_limits(0, 0) == 0
    assert lib.moe_gate_bwd(None, 4, 8, 4, 1, None, None, None, None, 0,
                            None) == _lib.MOE_EINVAL                # Epad < E
    # empty work is a no-op success
    assert lib.moe_topk_gate(None, 0, 0, 8, 1, None, None, None, None) == 0
    assert lib.moe_exclusive_scan_i64(None, 0, None, None, 0, None) == 0


def test_workspace_sizes():
    lib = _lib.load()
    T = (1000 + 127) // 128
    assert lib.moe_plan_workspace_bytes(1000, 16, 2) == (1000 * 2 + 2 * T * 16 + 16) * 4
    assert lib.moe_scan_workspace_bytes(10) >= 8
    assert lib.moe_scan_workspace_bytes(50_000_000) > lib.moe_scan_workspace_bytes(5000)


def test_gating_config_mirrors_reference():
    # test_gating.py:104-112 and :159-164
    for bad in [dict(num_experts=8, k=3), dict(num_experts=0, k=1),
                dict(num_experts=8, k=1, capacity_factor=0.0), dict(num_experts=1, k=2)]:
        with pytest.raises(ValueError):
            GatingConfig(**bad)
    assert GatingConfig(64, k=1, capacity_factor=1.0).capacity(512) == 8
    assert GatingConfig(64, k=1, capacity_factor=1.25).capacity(512) == 10
    assert GatingConfig(64, k=2, capacity_factor=1.0).capacity(512) == 16
    assert GatingConfig(4, k=1, capacity_factor=1e-9).capacity(8) == 1
    assert GatingConfig(4, k=1).capacity(0) == 0


def test_capacity_table_golden():
    z = np.load(os.path.join(ROOT, "tests", "golden", "plans.npz"))
    for e, k, cf, s, cap in z["capacity_table"]:
        assert GatingConfig(int(e), int(k), float(cf)).capacity(int(s)) == int(cap)


def test_layer_spec_validation():
    with pytest.raises(ValidationError):
        LayerSpec(kind="conv", hidden=8)
    with pytest.raises(ValidationError):
        LayerSpec(kind="moe", hidden=8, experts=2, gating=None)
    with pytest.raises(ValidationError):
        LayerSpec(kind="moe", hidden=8, experts=2, gating=GatingConfig(3))
    with pytest.raises(ValidationError):
        LayerSpec(kind="dense", hidden=8, experts=2)


def test_init_params_match_reference_draw_order():
    from oracle import moe_oracle as O

    spec = LayerSpec(kind="moe", hidden=8, experts=3, residual=True, gating=GatingConfig(3))
    p = init_layer_params(spec, np.random.default_rng(5))
    gw, experts, shared = O.init_layer_params(8, 3, True, np.random.default_rng(5))
    assert np.array_equal(p.gate_w.value, gw)
    for a, b in zip(p.experts, experts):
        assert np.array_equal(a.w1.value, b[0]) and np.array_equal(a.w2.value, b[2])
    assert np.array_equal(p.shared.w2.value, shared[2])


def test_no_cpu_fallback():
    import torch

    from paper_2201_05596_b200 import gating

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeUnavailable):
        gating.top_k_gate(np.zeros((4, 3)), GatingConfig(3))


def test_ctypes_signature_arity_matches_header():
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(rf"{name}\s*\(([^)]*)\)", text, flags=re.S)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name
    assert ctypes.sizeof(ctypes.c_void_p) == 8
