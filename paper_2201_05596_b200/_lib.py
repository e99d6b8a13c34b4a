"""ctypes binding of libmoe_b200.so (the C ABI in include/moe_b200.h).

There is no CPU fallback: if the shared library is missing or no sm_100 GPU
is present, every compute call raises. `load()` builds nothing; run
`python -m paper_2201_05596_b200.build` (or __graft_entry__.build()) first.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# MOE_B200_LIB: an alternative in-tree build (A/B tuning of compile-time variants)
LIB_PATH = os.environ.get("MOE_B200_LIB") or os.path.join(HERE, "libmoe_b200.so")

MOE_F32, MOE_BF16, MOE_F64 = 0, 1, 2
MOE_ACT_NONE, MOE_ACT_GELU = 0, 1
MOE_ACT_GELU_SAVE, MOE_ACT_GELU_BWD = 3, 4
MOE_GEMM_PAD_SCRATCH = 0x100  # act flag: rows past each group's count are scratch
MOE_GEMM_TILE256 = 0x200  # act flag: keep 256-column tiles
ROUTE_TILE = 128
MOE_EINVAL = -22

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_Z = ctypes.c_size_t

# name -> (restype, argtypes), mirroring include/moe_b200.h
SIGNATURES = {
    "moe_abi_version": (_I, []),
    "moe_topk_gate": (_I, [_P, _I, _L, _I, _I, _P, _P, _P, _P]),
    "moe_plan_tiles": (_I, [_P, _L, _I, _I, _P, _P, _P]),
    "moe_plan_scan": (_I, [_P, _L, _I, _L, _P, _P, _P, _P, _P]),
    "moe_plan_slots": (_I, [_P, _P, _P, _L, _I, _I, _L, _P, _P]),
    "moe_plan_workspace_bytes": (_Z, [_L, _I, _I]),
    "moe_build_plan": (_I, [_P, _L, _I, _I, _L, _P, _P, _P, _Z, _P]),
    "moe_scan_workspace_bytes": (_Z, [_L]),
    "moe_exclusive_scan_i64": (_I, [_P, _L, _P, _P, _Z, _P]),
    "moe_blelloch_scan_f64": (_I, [_P, _L, _P]),
    "moe_scatter": (_I, [_P, _L, _L, _I, _I, _L, _P, _P, _P, _P, _P]),
    "moe_dispatch": (_I, [_P, _L, _L, _I, _I, _L, _P, _P, _P, _P, _P, _P]),
    "moe_dispatch_ep": (_I, [_P, _L, _L, _I, _I, _L, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moe_dispatch_fused": (_I, [_P, _L, _L, _I, _I, _L, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moe_combine": (_I, [_P, _I, _L, _I, _I, _I, _L, _P, _P, _P, _P, _I, _P, _P, _P, _I, _P]),
    "moe_gate_gemm_bf16": (_I, [_P, _P, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "moe_gate_gemm_bf16_stats": (_I, [_P, _P, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "moe_load_balance_workspace_bytes": (_Z, [_I]),
    "moe_load_balance_loss": (_I, [_P, _L, _I, _I, _P, _I, _P, _P, _Z, _P]),
    "moe_load_balance_loss_from_stats": (_I, [_P, _P, _L, _I, _I, _P, _P]),
    "moe_grouped_gemm_bf16": (_I, [_P, _L, _I, _P, _L, _I, _P, _P, _I, _P, _L, _P, _L, _P, _L,
                                   _I, _P]),
    "moe_grouped_gemm_bf16_combine": (_I, [_P, _L, _I, _P, _L, _I, _P, _I, _P, _L, _P, _L, _P,
                                           _L, _P, _P, _P, _P, _P, _P]),
    "moe_enable_peer_access": (_I, [_I]),
    "moe_ipc_malloc": (_I, [_Z, _P]),
    "moe_ipc_free": (_I, [_P]),
    "moe_ipc_get_handle": (_I, [_P, _P]),
    "moe_ipc_open_handle": (_I, [_P, _P]),
    "moe_ipc_close_handle": (_I, [_P]),
    "moe_ep_plan": (_I, [_P, _I, _I, _I, _L, _P, _P, _P, _P, _P, _P]),
    "moe_ipc_barrier": (_I, [_P, _P, _I, _I, _P, _P, _P]),
    "moe_ipc_allgather_i32": (_I, [_P, _I, _P, _I, _I, _P, _P, _P, _P, _P]),
    "moe_dispatch_p2p": (_I, [_P, _L, _L, _I, _I, _L, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P,
                              _P, _P, _P, _I, _P]),
    "moe_grouped_gemm_bf16_push": (_I, [_P, _L, _I, _P, _L, _I, _P, _I, _P, _L, _P, _P, _L, _I,
                                        _P, _P, _P, _P, _P, _P]),
    "moe_ep_plan_padded": (_I, [_P, _I, _I, _I, _L, _P, _P, _P, _P, _P, _P]),
    "moe_grouped_gemm_bf16_combine_rows": (_I, [_P, _L, _I, _P, _L, _I, _P, _I, _P, _P, _P, _L,
                                                _P, _P, _P, _P, _P]),
    "moe_pull_rows_p2p": (_I, [_L, _L, _I, _I, _P, _P, _I, _P, _P, _P]),
    "moe_grouped_gemm_bf16_aux": (_I, [_P, _L, _I, _P, _L, _I, _P, _P, _I, _P, _L, _P, _L, _P, _L,
                                       _I, _P, _P]),
    "moe_combine_bwd_bf16": (_I, [_P, _P, _L, _I, _I, _I, _L, _P, _P, _P, _P, _P, _P]),
    "moe_gate_bwd": (_I, [_P, _L, _I, _I, _I, _P, _P, _P, _P, _I, _P]),
    "moe_gather_rows": (_I, [_P, _L, _P, _L, _P, _P]),
    "moe_ep_plan_chunked": (_I, [_P, _I, _I, _I, _I, _L, _P, _P, _P, _P, _P, _P]),
    "moe_set_launch_limits": (_I, [_I, _I]),
    "moe_grouped_gemm_bf16_gather": (_I, [_P, _L, _P, _I, _P, _L, _I, _P, _P, _I, _L, _P, _L, _L,
                                          _I, _P]),
    "moe_colsum_rows_bf16": (_I, [_P, _I, _I, _L, _P, _L, _P, _P]),
    "moe_grouped_gemm_bf16_wgrad": (_I, [_P, _L, _I, _P, _I, _I, _L, _P, _L, _P, _P]),
    "moe_gemm_bf16_wgrad_f32": (_I, [_P, _L, _I, _P, _I, _P, _P]),
    "moe_bwd_dx_bf16": (_I, [_P, _P, _L, _I, _I, _I, _L, _P, _P, _P, _P, _P, _P]),
    "moe_grouped_gemm_f32": (_I, [_P, _I, _P, _I, _P, _P, _I, _P, _L, _P, _L, _P, _L, _I, _P]),
    "moe_residual_gemm_bf16": (_I, [_P, _L, _P, _L, _I, _I, _P, _L, _I, _P, _P, _I, _L, _P, _P, _L,
                                    _I, _I, _P, _P, _P, _I, _L, _P, _P, _L, _P, _P]),
}

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    """The CUDA extension (or an sm_100 device) is missing; no fallback exists."""


def load():
    """Load (once) and return the ctypes handle; raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} not built; run `python -m paper_2201_05596_b200.build`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.moe_abi_version() != 1:
                raise NativeUnavailable("libmoe_b200.so ABI version mismatch")
            _lib = lib
    return _lib


def require_device(t: torch.Tensor | None = None) -> torch.device:
    """The B200 path needs a CUDA sm_100 device; raise loudly otherwise."""
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 MoE path has no CPU fallback")
    dev = t.device if (t is not None and t.is_cuda) else torch.device("cuda", torch.cuda.current_device())
    major, _ = torch.cuda.get_device_capability(dev)
    if major != 10:
        raise NativeUnavailable(f"device {dev} is sm_{major}x; kernels are built for sm_100a")
    load()
    return dev


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def check(rc: int, what: str) -> None:
    if rc == MOE_EINVAL:
        raise ValueError(f"{what}: invalid arguments (MOE_EINVAL)")
    if rc != 0:
        raise RuntimeError(f"{what} failed with code {rc}")


def call(name: str, *args) -> None:
    lib = load()
    _count(name)
    check(getattr(lib, name)(*args), name)


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return MOE_F32
    if dt == torch.bfloat16:
        return MOE_BF16
    if dt == torch.float64:
        return MOE_F64
    raise TypeError(f"unsupported dtype {dt}")


# ---------------------------------------------------------------------------
# instrumentation: kernel-launch counter and per-phase CUDA-event timer
# ---------------------------------------------------------------------------

_NON_LAUNCH = {"moe_abi_version", "moe_plan_workspace_bytes", "moe_scan_workspace_bytes",
               "moe_enable_peer_access",
               "moe_load_balance_workspace_bytes",
               "moe_ipc_malloc", "moe_ipc_free", "moe_ipc_get_handle", "moe_ipc_open_handle",
               "moe_ipc_close_handle"}
# entry points that launch more than one kernel per call
_MULTI = {"moe_build_plan": 3}
_launches = 0


def launch_count() -> int:
    """Number of kernel launches issued through this binding (per process)."""
    return _launches


def _count(name: str) -> None:
    global _launches
    if name not in _NON_LAUNCH:
        _launches += _MULTI.get(name, 1)


class PhaseTimer:
    """CUDA events around named phases on the current stream; no host sync
    inside the timed region (events are read after the caller synchronizes)."""

    def __init__(self) -> None:
        self.rec: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    def start(self, name: str):
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        return (name, e0)

    def stop(self, tok) -> None:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self.rec.append((tok[0], tok[1], e1))

    def summary(self, steps: int) -> dict:
        out: dict[str, float] = {}
        for name, a, b in self.rec:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return {k: v / max(steps, 1) for k, v in out.items()}
