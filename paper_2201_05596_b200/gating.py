"""Top-k routing with capacity-slotted dispatch tables, on the B200.

Drop-in for ``moekit.gating`` (reference ``gating.py``; public names from
gating.py:36-50). Same dataclasses, field names, argument order, validation
and exceptions; the bodies launch the sm_100a kernels of libmoe_b200.so:

  top_k_gate           -> moe_topk_gate         (gating.py:142-163)
  exclusive_scan_blelloch -> moe_exclusive_scan_i64 / moe_blelloch_scan_f64
                                                 (gating.py:171-203)
  build_dispatch_plan  -> moe_build_plan        (gating.py:211-247)
  scatter_tokens       -> moe_scatter           (gating.py:255-278)
  combine_tokens       -> moe_combine           (gating.py:281-307)

Inputs may be NumPy arrays (results come back as NumPy with the reference's
dtypes: int64 ids/slots, float64 probabilities and buffers) or torch CUDA
tensors (results stay on the device; routing tables are int32 there).
NumPy float64 data stays float64 on the device, so scatter is an exact copy
and combine reproduces NumPy's rounding bit for bit. There is no CPU path:
without the CUDA extension every call raises.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .tensor import ShapeError

__all__ = [
    "DROPPED",
    "GatingConfig",
    "TopKGate",
    "DispatchPlan",
    "ExpertBuffers",
    "OpCounter",
    "top_k_gate",
    "exclusive_scan_blelloch",
    "build_dispatch_plan",
    "scatter_tokens",
    "combine_tokens",
]

DROPPED = -1  # gating.py:52


@dataclass(frozen=True)
class GatingConfig:
    """Routing hyperparameters (gating.py:55-80)."""

    num_experts: int
    k: int = 1
    capacity_factor: float = 1.0

    def __post_init__(self) -> None:
        if self.num_experts < 1:
            raise ValueError(f"num_experts must be >= 1, got {self.num_experts}")
        if self.k not in (1, 2):
            raise ValueError(f"k must be 1 or 2, got {self.k}")
        if self.k > self.num_experts:
            raise ValueError(f"k={self.k} exceeds num_experts={self.num_experts}")
        if not (self.capacity_factor > 0):
            raise ValueError(f"capacity_factor must be positive, got {self.capacity_factor}")

    def capacity(self, num_tokens: int) -> int:
        """ceil(cf * S * k / E) in float64, evaluated left to right (gating.py:77-80)."""
        if num_tokens == 0:
            return 0
        return int(np.ceil(self.capacity_factor * num_tokens * self.k / self.num_experts))


@dataclass(frozen=True)
class TopKGate:
    expert_ids: object  # (S, k)
    gate_probs: object  # (S, k)
    probs: object       # (S, E)


@dataclass(frozen=True)
class DispatchPlan:
    num_tokens: int
    num_experts: int
    k: int
    capacity: int
    expert_ids: object
    gate_probs: object
    slots: object
    expert_load: object

    def kept_mask(self):
        return self.slots != DROPPED


@dataclass
class ExpertBuffers:
    data: object      # (E, capacity, M)
    occupied: object  # (E, capacity) bool


@dataclass
class OpCounter:
    """Routing-transform op counter; convention S*c*M per transform (gating.py:127-134)."""

    ops: int = 0

    def add(self, n: int) -> None:
        self.ops += int(n)


# ---------------------------------------------------------------------------
# host <-> device plumbing
# ---------------------------------------------------------------------------


def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def _dev(x, dtype: torch.dtype | None = None) -> torch.Tensor:
    dev = _lib.require_device(x if _is_torch(x) else None)
    t = x if _is_torch(x) else torch.from_numpy(np.ascontiguousarray(x))
    t = t.to(device=dev, dtype=dtype if dtype is not None else t.dtype, non_blocking=False)
    return t.contiguous()


def _host(t: torch.Tensor, np_dtype) -> np.ndarray:
    return t.detach().cpu().numpy().astype(np_dtype, copy=False)


def _shape(x) -> tuple:
    return tuple(x.shape)


# ---------------------------------------------------------------------------
# gating
# ---------------------------------------------------------------------------


def top_k_gate(logits, cfg: GatingConfig) -> TopKGate:
    """Each token's k highest-logit experts; probabilities are the full-E
    softmax at the chosen ids, not renormalised; ties break to the lower
    expert index (gating.py:142-163)."""
    as_np = not _is_torch(logits)
    if as_np:
        logits = np.asarray(logits, dtype=np.float64)
    if len(_shape(logits)) != 2:
        raise ShapeError(f"gate logits must be 2-D, got shape {_shape(logits)}")
    s, e = _shape(logits)
    if e != cfg.num_experts:
        raise ShapeError(f"gate logits have {e} columns, config expects {cfg.num_experts}")
    if as_np:
        lg = _dev(logits, torch.float64)
    else:
        lg = _dev(logits)
        if lg.dtype not in (torch.float32, torch.float64):
            lg = lg.float()
    dev = lg.device
    ids = torch.empty((s, cfg.k), dtype=torch.int32, device=dev)
    gp = torch.empty((s, cfg.k), dtype=lg.dtype, device=dev)
    probs = torch.empty((s, e), dtype=lg.dtype, device=dev)
    if s:
        _lib.call("moe_topk_gate", lg.data_ptr(), _lib.dtype_code(lg.dtype), s, e, cfg.k,
                  ids.data_ptr(), gp.data_ptr(), probs.data_ptr(), _lib.stream_ptr())
    if as_np:
        return TopKGate(expert_ids=_host(ids, np.int64), gate_probs=_host(gp, np.float64),
                        probs=_host(probs, np.float64))
    return TopKGate(expert_ids=ids, gate_probs=gp, probs=probs)


def exclusive_scan_blelloch(values):
    """Exclusive prefix sum with the work-efficient tree (gating.py:171-203).

    Integer/bool input -> exact int64 scan on the device. Float input ->
    float64 up-sweep/down-sweep over the zero-padded power-of-two buffer, the
    reference's own association order, so results are bitwise identical."""
    as_np = not _is_torch(values)
    v = np.asarray(values) if as_np else values
    if v.ndim != 1:
        raise ShapeError(f"scan input must be 1-D, got shape {tuple(v.shape)}")
    n = v.shape[0]
    is_int = (v.dtype.kind in "iub") if as_np else (not v.dtype.is_floating_point)
    if n == 0:
        if as_np:
            return np.zeros(0, dtype=np.int64 if is_int else v.dtype)
        return torch.zeros(0, dtype=torch.int64 if is_int else v.dtype, device=v.device)
    if is_int:
        src = _dev(v.astype(np.int64) if as_np else v.to(torch.int64), torch.int64)
        out = torch.empty(n, dtype=torch.int64, device=src.device)
        lib = _lib.load()
        wsb = lib.moe_scan_workspace_bytes(n)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=src.device)
        _lib.call("moe_exclusive_scan_i64", src.data_ptr(), n, out.data_ptr(), ws.data_ptr(), wsb,
                  _lib.stream_ptr())
        return _host(out, np.int64) if as_np else out
    m = 1 << (n - 1).bit_length()
    src = _dev(v.astype(np.float64) if as_np else v.to(torch.float64), torch.float64)
    tree = torch.zeros(m, dtype=torch.float64, device=src.device)
    tree[:n] = src
    _lib.call("moe_blelloch_scan_f64", tree.data_ptr(), m, _lib.stream_ptr())
    return _host(tree[:n], np.float64) if as_np else tree[:n]


def _route_ids(expert_ids, num_experts: int):
    """int32 ids for the device; an id outside [0, E) matches no expert's
    indicator in the reference (gating.py:229-230) and stays DROPPED, so it is
    mapped to -1 here (before the int32 narrowing could alias it)."""
    if _is_torch(expert_ids):
        ids = expert_ids.to(torch.int64)
        return torch.where((ids >= 0) & (ids < num_experts), ids, -1).to(torch.int32)
    ids = np.asarray(expert_ids, dtype=np.int64)
    return np.where((ids >= 0) & (ids < num_experts), ids, -1).astype(np.int32)


def build_dispatch_plan(gates: TopKGate, cfg: GatingConfig, num_tokens: int) -> DispatchPlan:
    """Capacity slots in flattened token-major order, DROPPED past capacity
    (gating.py:211-247). Bit-exact with the reference for any ids."""
    if tuple(gates.expert_ids.shape) != (num_tokens, cfg.k):
        raise ShapeError(
            f"gate table shape {tuple(gates.expert_ids.shape)} does not match "
            f"({num_tokens}, {cfg.k})")
    as_np = not _is_torch(gates.expert_ids)
    cap = cfg.capacity(num_tokens)
    ids = _dev(_route_ids(gates.expert_ids, cfg.num_experts), torch.int32)
    dev = ids.device
    slots = torch.empty((num_tokens, cfg.k), dtype=torch.int32, device=dev)
    load = torch.empty(cfg.num_experts, dtype=torch.int32, device=dev)
    lib = _lib.load()
    wsb = lib.moe_plan_workspace_bytes(num_tokens, cfg.num_experts, cfg.k)
    ws = torch.empty(max(wsb, 4), dtype=torch.uint8, device=dev)
    _lib.call("moe_build_plan", ids.data_ptr(), num_tokens, cfg.num_experts, cfg.k, cap,
              slots.data_ptr(), load.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr())
    if as_np:
        return DispatchPlan(num_tokens=num_tokens, num_experts=cfg.num_experts, k=cfg.k,
                            capacity=cap, expert_ids=np.array(gates.expert_ids, copy=True),
                            gate_probs=np.array(gates.gate_probs, copy=True),
                            slots=_host(slots, np.int64), expert_load=_host(load, np.int64))
    return DispatchPlan(num_tokens=num_tokens, num_experts=cfg.num_experts, k=cfg.k,
                        capacity=cap, expert_ids=gates.expert_ids.clone(),
                        gate_probs=gates.gate_probs.clone(), slots=slots, expert_load=load)


def _plan_tables(plan: DispatchPlan, dev) -> tuple[torch.Tensor, torch.Tensor]:
    ids = _dev(np.asarray(plan.expert_ids, dtype=np.int32) if not _is_torch(plan.expert_ids)
               else plan.expert_ids, torch.int32)
    slots = _dev(np.asarray(plan.slots, dtype=np.int32) if not _is_torch(plan.slots)
                 else plan.slots, torch.int32)
    ids, slots = ids.to(dev), slots.to(dev)
    # a kept assignment must address a real (expert, slot) row: the reference's
    # fancy indexing raises on anything else (gating.py:271-275, :298-304)
    kept = slots != DROPPED
    bad = kept & ((ids < 0) | (ids >= plan.num_experts) | (slots < 0) |
                  (slots >= plan.capacity))
    if bool(bad.any()):
        raise IndexError("plan has a kept assignment outside the (num_experts, capacity) buffers")
    return ids, slots


def scatter_tokens(batch, plan: DispatchPlan, counter: OpCounter | None = None) -> ExpertBuffers:
    """data[e, slot] = batch[t] for kept assignments, unoccupied slots zero
    (gating.py:255-278). Exact row copies in the input dtype."""
    as_np = not _is_torch(batch)
    if as_np:
        batch = np.asarray(batch, dtype=np.float64)
    if len(_shape(batch)) != 2 or _shape(batch)[0] != plan.num_tokens:
        raise ShapeError(f"batch shape {_shape(batch)} does not match plan S={plan.num_tokens}")
    m = _shape(batch)[1]
    x = _dev(batch)
    dev = x.device
    data = torch.zeros((plan.num_experts, plan.capacity, m), dtype=x.dtype, device=dev)
    occ = torch.zeros((plan.num_experts, plan.capacity), dtype=torch.uint8, device=dev)
    if plan.num_tokens and plan.capacity and m:
        ids, slots = _plan_tables(plan, dev)
        _lib.call("moe_scatter", x.data_ptr(), plan.num_tokens, m * x.element_size(),
                  plan.num_experts, plan.k, plan.capacity, ids.data_ptr(), slots.data_ptr(),
                  data.data_ptr(), occ.data_ptr(), _lib.stream_ptr())
    if counter is not None:
        counter.add(plan.num_tokens * plan.capacity * m)
    if as_np:
        return ExpertBuffers(data=_host(data, np.float64), occupied=_host(occ, bool))
    return ExpertBuffers(data=data, occupied=occ.bool())


def combine_tokens(outputs, plan: DispatchPlan, counter: OpCounter | None = None):
    """out[t] = sum over kept assignments of gate_prob * data[e, slot], in
    token-major order; fully dropped tokens give zero rows (gating.py:281-307).
    ``outputs`` is duck-typed on ``.data`` (tests/test_gating.py:351-356)."""
    data = outputs.data
    as_np = not _is_torch(data)
    if as_np:
        data = np.asarray(data, dtype=np.float64)
    e_count, cap, m = _shape(data)
    if e_count != plan.num_experts or cap != plan.capacity:
        raise ShapeError(
            f"buffer shape {_shape(data)} does not match plan "
            f"(E={plan.num_experts}, c={plan.capacity})")
    y = _dev(data)
    dev = y.device
    if y.dtype == torch.float64:
        gp_dtype = torch.float64
    elif y.dtype in (torch.float32, torch.bfloat16):
        gp_dtype = torch.float32
    else:
        raise TypeError(f"unsupported buffer dtype {y.dtype}")
    out = torch.zeros((plan.num_tokens, m), dtype=y.dtype, device=dev)
    if plan.num_tokens and m:
        ids, slots = _plan_tables(plan, dev)
        gp = _dev(np.asarray(plan.gate_probs) if not _is_torch(plan.gate_probs)
                  else plan.gate_probs, gp_dtype)
        _lib.call("moe_combine", y.data_ptr(), _lib.dtype_code(y.dtype), plan.num_tokens, m,
                  plan.num_experts, plan.k, plan.capacity, ids.data_ptr(), slots.data_ptr(), None,
                  gp.data_ptr(), _lib.dtype_code(gp_dtype), None, None, out.data_ptr(), 0,
                  _lib.stream_ptr())
    if counter is not None:
        counter.add(plan.num_tokens * plan.capacity * m)
    return _host(out, np.float64) if as_np else out
