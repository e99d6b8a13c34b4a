"""MoE layer forward on the B200: drop-in for the layer half of ``moekit.arch``.

Reference: arch.py:65-96 (FFN_MULT, LayerSpec), arch.py:316-413 (FfnParams,
MoeLayerParams, init_layer_params, forward_ffn, forward_layer). Same names,
fields, validation and exceptions. The forward is inference-only (no tape):
the reference's tape-aware training use (arch.py:375-377) is out of scope.

Two device paths, chosen by the activation dtype:

* bf16 (the performance path): tcgen05 gate GEMM with the routing epilogue
  -> capacity scan -> dispatch (slots fused) -> grouped tcgen05 GEMM1
  (bias + tanh-GELU) -> grouped GEMM2 (bias) -> combine (+x, +shared MLP).
* fp32 (the parity path for BASELINE config 1; NumPy inputs use it): the same
  pipeline with an fp32 SIMT grouped GEMM and an accurate tanhf GELU.

``MoeLayer`` holds the packed device weights (bf16 weights transposed to
K-major for the tensor cores, fp32 biases) plus reusable workspaces; build it
once and call it. ``forward_layer(x, spec, params)`` accepts either a
``MoeLayer`` or reference-style ``MoeLayerParams`` (packed on every call).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .gating import GatingConfig
from .tensor import ShapeError, Tensor, as_array

__all__ = [
    "ValidationError",
    "FFN_MULT",
    "LayerSpec",
    "FfnParams",
    "MoeLayerParams",
    "init_layer_params",
    "forward_ffn",
    "forward_layer",
    "MoeLayer",
    "DenseFfn",
    "load_balance_loss",
]

FFN_MULT = 4  # arch.py:65


class ValidationError(ValueError):
    """Structurally invalid layer description (arch.py:68)."""


@dataclass(frozen=True)
class LayerSpec:
    """One transformer block's feed-forward slot (arch.py:72-96)."""

    kind: str
    hidden: int
    experts: int = 0
    residual: bool = False
    gating: GatingConfig | None = None

    def __post_init__(self) -> None:
        if self.kind not in ("dense", "moe"):
            raise ValidationError(f"unknown layer kind {self.kind!r}")
        if self.hidden < 1:
            raise ValidationError("hidden width must be positive")
        if self.kind == "moe":
            if self.experts < 1:
                raise ValidationError("moe layer needs at least one expert")
            if self.gating is None:
                raise ValidationError("moe layer needs a gating config")
            if self.gating.num_experts != self.experts:
                raise ValidationError("gating config expert count mismatch")
        else:
            if self.experts != 0 or self.gating is not None or self.residual:
                raise ValidationError("dense layer cannot carry expert fields")


@dataclass
class FfnParams:
    """w1 (M, 4M), b1 (1, 4M), w2 (4M, M), b2 (1, M) (arch.py:321-329)."""

    w1: object
    b1: object
    w2: object
    b2: object

    def leaves(self) -> list:
        return [self.w1, self.b1, self.w2, self.b2]


@dataclass
class MoeLayerParams:
    """gate_w (M, E), experts, optional shared MLP (arch.py:332-344)."""

    gate_w: object
    experts: tuple
    shared: FfnParams | None = None

    def leaves(self) -> list:
        out = [self.gate_w]
        for e in self.experts:
            out.extend(e.leaves())
        if self.shared is not None:
            out.extend(self.shared.leaves())
        return out


def _init_ffn(m: int, rng: np.random.Generator, scale: float) -> FfnParams:
    inner = FFN_MULT * m
    return FfnParams(
        w1=Tensor(rng.standard_normal((m, inner)) * scale),
        b1=Tensor(np.zeros((1, inner))),
        w2=Tensor(rng.standard_normal((inner, m)) * scale),
        b2=Tensor(np.zeros((1, m))),
    )


def init_layer_params(spec: LayerSpec, rng: np.random.Generator, scale: float = 0.1):
    """Host parameters with the reference's draw order (arch.py:347-365), so a
    seeded rng gives the same weights as ``moekit.arch.init_layer_params``."""
    if spec.kind == "dense":
        return _init_ffn(spec.hidden, rng, scale)
    return MoeLayerParams(
        gate_w=Tensor(rng.standard_normal((spec.hidden, spec.experts)) * scale),
        experts=tuple(_init_ffn(spec.hidden, rng, scale) for _ in range(spec.experts)),
        shared=_init_ffn(spec.hidden, rng, scale) if spec.residual else None,
    )


# ---------------------------------------------------------------------------
# packing
# ---------------------------------------------------------------------------


def _t(x, dev, dtype) -> torch.Tensor:
    x = as_array(x)
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype)
    return torch.as_tensor(np.asarray(x), device=dev).to(dtype)


def _check_dtype(dtype: torch.dtype) -> torch.dtype:
    if dtype not in (torch.bfloat16, torch.float32):
        raise TypeError(f"layer dtype must be torch.bfloat16 or torch.float32, got {dtype}")
    return dtype


class DenseFfn:
    """One packed FFN (the shared Residual-MoE MLP or a dense layer) on device."""

    def __init__(self, p: FfnParams, hidden: int, dtype: torch.dtype, dev) -> None:
        self.dtype, self.M, self.F = dtype, hidden, FFN_MULT * hidden
        w1, w2 = _t(p.w1, dev, torch.float32), _t(p.w2, dev, torch.float32)
        if tuple(w1.shape) != (self.M, self.F) or tuple(w2.shape) != (self.F, self.M):
            raise ShapeError(f"ffn weights {tuple(w1.shape)}/{tuple(w2.shape)} do not match "
                             f"hidden {hidden}")
        self.b1 = _t(p.b1, dev, torch.float32).reshape(1, self.F).contiguous()
        self.b2 = _t(p.b2, dev, torch.float32).reshape(1, self.M).contiguous()
        if dtype == torch.bfloat16:  # W^T, K-major for tcgen05
            self.w1 = w1.t().contiguous().to(dtype)
            self.w2 = w2.t().contiguous().to(dtype)
        else:
            self.w1, self.w2 = w1.contiguous(), w2.contiguous()

    def __call__(self, x: torch.Tensor, h: torch.Tensor | None = None,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        s = x.shape[0]
        h = torch.empty((s, self.F), dtype=self.dtype, device=x.device) if h is None else h
        out = torch.empty((s, self.M), dtype=self.dtype, device=x.device) if out is None else out
        _grouped_gemm(self.dtype, x, s, self.M, self.w1, self.F, self.b1, h, 1, None, 0, None, s,
                      s, _lib.MOE_ACT_GELU, scratch_pad=True)
        _grouped_gemm(self.dtype, h, s, self.F, self.w2, self.M, self.b2, out, 1, None, 0, None, s,
                      s, _lib.MOE_ACT_NONE, scratch_pad=True)
        return out


class _Phases:
    """Optional per-phase CUDA-event timing (bench.py); a no-op without a timer."""

    def __init__(self, timer) -> None:
        self.timer, self.tok = timer, None

    def __call__(self, name) -> None:
        if self.timer is None:
            return
        if self.tok is not None:
            self.timer.stop(self.tok)
        self.tok = self.timer.start(name) if name else None


def _grouped_gemm(dtype, a, a_rows, K, w, N, bias, d, G, row_start, row_stride, rows, rows_const,
                  max_rows, act, scratch_pad=False):
    """scratch_pad: rows past each group's count (up to row_stride) are padding
    the kernel may overwrite, which lets the bf16 epilogue use TMA tensor stores."""
    st = _lib.stream_ptr()
    if dtype == torch.bfloat16:
        if scratch_pad:
            act |= _lib.MOE_GEMM_PAD_SCRATCH
        _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), a_rows, K, w.data_ptr(),
                  w.numel() // K, N, _lib.ptr(bias), d.data_ptr(), G, _lib.ptr(row_start),
                  row_stride, _lib.ptr(rows), rows_const, None, max_rows, act, st)
    else:
        _lib.call("moe_grouped_gemm_f32", a.data_ptr(), K, w.data_ptr(), N, _lib.ptr(bias),
                  d.data_ptr(), G, _lib.ptr(row_start), row_stride, _lib.ptr(rows), rows_const,
                  None, max_rows, act, st)


class MoeLayer:
    """A Standard / Residual (PR-MoE) MoE layer packed for the B200.

    Device layout (HBM): gate weight (bf16: W_g^T zero-padded to Epad rows;
    fp32: W_g as (M, E)); expert weights stacked per expert (bf16: W1^T as
    (E*F, M) and W2^T as (E*M, F), K-major; fp32: (E, M, F) and (E, F, M));
    biases fp32 (E, F) / (E, M). Activations (S, M) row-major.
    """

    def __init__(self, spec: LayerSpec, params: MoeLayerParams, dtype=torch.bfloat16,
                 device=None, fuse_combine: bool = True, aux_loss: bool = False,
                 gather_rows: bool = False) -> None:
        if spec.kind != "moe":
            raise ValidationError("MoeLayer needs a moe LayerSpec")
        dev = _lib.require_device(None) if device is None else torch.device(device)
        _lib.load()
        self.spec, self.dtype, self.device = spec, _check_dtype(dtype), dev
        M, E = spec.hidden, spec.experts
        F = FFN_MULT * M
        self.M, self.E, self.F, self.k = M, E, F, spec.gating.k
        if len(params.experts) != E:
            raise ShapeError(f"{len(params.experts)} experts given, spec has {E}")
        gw = _t(params.gate_w, dev, torch.float32)
        if tuple(gw.shape) != (M, E):
            raise ShapeError(f"gate_w shape {tuple(gw.shape)} != ({M}, {E})")
        w1 = torch.stack([_t(p.w1, dev, torch.float32) for p in params.experts])
        w2 = torch.stack([_t(p.w2, dev, torch.float32) for p in params.experts])
        if tuple(w1.shape) != (E, M, F) or tuple(w2.shape) != (E, F, M):
            raise ShapeError("expert weight shapes do not match the spec")
        self.b1 = torch.stack([_t(p.b1, dev, torch.float32).reshape(F) for p in params.experts])
        self.b2 = torch.stack([_t(p.b2, dev, torch.float32).reshape(M) for p in params.experts])
        # E > 256 (beyond one tcgen05 N tile of the fused gate): logits from the fp32
        # grouped GEMM on the bf16-rounded x and W_g, then the stand-alone top-k /
        # plan-tiles kernels, as on the fp32 path; the expert GEMMs stay tcgen05
        self.wide_gate = self.dtype == torch.bfloat16 and E > 256
        if self.dtype == torch.bfloat16:
            if M % 8:
                raise ValueError("the bf16 tensor-core path needs hidden % 8 == 0")
            self.epad = max(32, 1 << (E - 1).bit_length())
            if self.wide_gate:
                self.wg = None
                self.wg32 = gw.to(torch.bfloat16).float().contiguous()  # (M, E)
            else:
                wg_t = torch.zeros((self.epad, M), dtype=torch.bfloat16, device=dev)
                wg_t[:E] = gw.t().to(torch.bfloat16)
                self.wg = wg_t
            self.w1 = w1.transpose(1, 2).reshape(E * F, M).contiguous().to(torch.bfloat16)
            self.w2 = w2.transpose(1, 2).reshape(E * M, F).contiguous().to(torch.bfloat16)
        else:
            self.wg = gw.contiguous()
            self.w1, self.w2 = w1.contiguous(), w2.contiguous()
        del w1, w2
        self.shared = (DenseFfn(params.shared, M, self.dtype, dev)
                       if (spec.residual and params.shared is not None) else None)
        if spec.residual and params.shared is None:
            raise ValidationError("residual layer needs shared MLP params")
        # bf16 Residual-MoE: the shared MLP runs as extra groups (weight index E) of the
        # expert GEMM launches and its GEMM2 epilogue does the combine + both residual
        # adds (moe_residual_gemm_bf16); the expert and shared weights live in one
        # stacked buffer, the DenseFfn / per-expert tensors are views into it
        self.grouped_shared = self.dtype == torch.bfloat16 and self.shared is not None
        if self.grouped_shared:
            sh = self.shared
            self.w1_all = torch.cat([self.w1, sh.w1]).contiguous()
            self.w2_all = torch.cat([self.w2, sh.w2]).contiguous()
            self.b1_all = torch.cat([self.b1, sh.b1]).contiguous()
            self.b2_all = torch.cat([self.b2, sh.b2]).contiguous()
            self.w1, self.w2 = self.w1_all[:E * F], self.w2_all[:E * M]
            self.b1, self.b2 = self.b1_all[:E], self.b2_all[:E]
            sh.w1, sh.w2 = self.w1_all[E * F:], self.w2_all[E * M:]
            sh.b1, sh.b2 = self.b1_all[E:], self.b2_all[E:]
        # k=1 bf16 layers without a shared MLP fold combine + residual into GEMM2
        self.fused_combine = bool(fuse_combine and self.dtype == torch.bfloat16 and
                                  self.k == 1 and self.shared is None)
        # gather_rows: GEMM1 gathers its A rows straight from x (TMA gather4) and
        # dispatch only routes. Bit-identical, but measured 2.3x slower for GEMM1 at
        # C3 (32 gather4 TMA ops per 16 KB stage, re-issued for every n-block), so the
        # dispatched copy (one 0.1 ms pass) stays the default.
        self.gather_rows = bool(gather_rows and self.fused_combine)
        self._ws: dict = {}
        self._pipe = None
        self.aux_loss = aux_loss

    # -- workspace -----------------------------------------------------------
    def workspace(self, S: int) -> dict:
        ws = self._ws.get(S)
        if ws is not None:
            return ws
        if len(self._ws) >= 4:  # keep a few batch sizes (e.g. prefill + decode) resident
            self._ws.pop(next(iter(self._ws)))
        dev, dt, E, M, F, k = self.device, self.dtype, self.E, self.M, self.F, self.k
        cap = self.spec.gating.capacity(S)
        T = (S + _lib.ROUTE_TILE - 1) // _lib.ROUTE_TILE
        i32 = dict(dtype=torch.int32, device=dev)
        # shared MLP grouped with the experts: its S tokens as ceil(S/cap) groups of
        # cap rows (needs groups of at least one 128-row tile and <= 2048 groups)
        nsh = -(-S // cap) if cap else 0
        grouped = bool(self.grouped_shared and cap >= 128 and E + nsh <= 2048)
        ws = dict(
            cap=cap, T=T, grouped_shared=grouped,
            ids=torch.empty((S, k), **i32), slots=torch.empty((S, k), **i32),
            local_rank=torch.empty((S, k), **i32),
            gp=torch.empty((S, k), dtype=torch.float32, device=dev),
            tile_counts=torch.empty((max(T, 1), E), **i32),
            tile_offsets=torch.empty((max(T, 1), E), **i32),
            totals=torch.empty(E, **i32), load=torch.empty(E, **i32),
            xbuf=(None if self.gather_rows else
                  torch.empty((max(E * cap, 1), M), dtype=dt, device=dev)),
            h=torch.empty((max(E * cap, 1), F), dtype=dt, device=dev),
            y=torch.empty((max(E * cap, 1), M), dtype=dt, device=dev),
        )
        if dt == torch.float32 or self.wide_gate:
            ws["logits"] = torch.empty((S, E), dtype=torch.float32, device=dev)
        ws["probsum"] = torch.zeros(E, dtype=torch.float32, device=dev)
        ws["aux"] = torch.zeros(1, dtype=torch.float64, device=dev)
        if self.fused_combine:
            ws["row_token"] = torch.empty(max(E * cap, 1), **i32)
            ws["row_prob"] = torch.empty(max(E * cap, 1), dtype=torch.float32, device=dev)
        if grouped:
            G = E + nsh
            rows_all = torch.empty(G, **i32)
            rows_all[E:] = torch.tensor([min(cap, S - j * cap) for j in range(nsh)], **i32)
            ws.update(G=G, rows_all=rows_all, load=rows_all[:E],
                      widx=torch.tensor(list(range(E)) + [E] * nsh, **i32),
                      h=torch.empty((G * cap, F), dtype=dt, device=dev))
        elif self.shared is not None:
            ws["hs"] = torch.empty((S, F), dtype=dt, device=dev)
            if dt == torch.float32:
                ws["ys"] = torch.empty((S, M), dtype=dt, device=dev)
            else:  # the shared GEMM2 + combine epilogue over one group of S token rows
                ws["sh_rows"] = torch.tensor([S], **i32)
                ws["sh_w"] = torch.zeros(1, **i32)
        self._ws[S] = ws
        return ws

    # -- forward ---------------------------------------------------------------
    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None,
                 logits_out: torch.Tensor | None = None, timer=None) -> torch.Tensor:
        return self.forward(x, out, logits_out, timer)

    # load-balance loss of the last forward (arch.py:297-313), when aux_loss=True:
    # the fused gate accumulates the softmax column sums, the plan scan the counts
    aux_loss: bool = False
    last_aux_loss: torch.Tensor | None = None

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None,
                logits_out: torch.Tensor | None = None, timer=None) -> torch.Tensor:
        """out = x + combine(experts(dispatch(x))) [+ shared MLP(x)]
        (arch.py:372-392). ``logits_out`` (S, E) fp32 receives the gate logits
        the routing decided on (the parity tests feed them to the oracle).

        A host ``x`` streams through ``pipeline.HostPipeline`` (async H2D /
        forward / D2H on separate streams, double-buffered); the result is a
        host tensor valid after the next device synchronisation."""
        if x.dim() != 2 or x.shape[1] != self.M:
            raise ShapeError(f"batch width {tuple(x.shape)} does not match layer hidden {self.M}")
        if not x.is_cuda:
            if self._pipe is None:
                from .pipeline import HostPipeline

                self._pipe = HostPipeline(self._forward_dev, self.M, self.dtype, self.device)
            xh = x if x.dtype == self.dtype else x.to(self.dtype)
            oh = out if (out is not None and not out.is_cuda) else None
            with torch.cuda.device(self.device):
                return self._pipe(xh, oh, logits_out=logits_out, timer=timer)
        # kernels launch on the current device: make it this layer's (one process
        # may drive layers on several GPUs)
        with torch.cuda.device(self.device):
            return self._forward_dev(x, out, logits_out, timer)

    def _forward_dev(self, x: torch.Tensor, out: torch.Tensor | None = None,
                     logits_out: torch.Tensor | None = None, timer=None) -> torch.Tensor:
        if x.device != self.device:
            x = x.to(device=self.device, non_blocking=True)
        if x.dtype != self.dtype:
            x = x.to(self.dtype)
        x = x.contiguous()
        S = x.shape[0]
        out = torch.empty_like(x) if out is None else out
        if S == 0:
            return out
        ws = self.workspace(S)
        cap, E, M, F, k = ws["cap"], self.E, self.M, self.F, self.k
        st = _lib.stream_ptr()
        ids, gp, lr, tc = ws["ids"], ws["gp"], ws["local_rank"], ws["tile_counts"]
        ph = _Phases(timer)
        ph("gate")
        aux = self.aux_loss
        if self.dtype == torch.bfloat16 and not self.wide_gate:
            if aux:
                ws["probsum"].zero_()
                _lib.call("moe_gate_gemm_bf16_stats", x.data_ptr(), self.wg.data_ptr(), S, M, E,
                          k, _lib.ptr(logits_out), ids.data_ptr(), gp.data_ptr(), lr.data_ptr(),
                          tc.data_ptr(), ws["probsum"].data_ptr(), st)
            else:
                _lib.call("moe_gate_gemm_bf16", x.data_ptr(), self.wg.data_ptr(), S, M, E, k,
                          _lib.ptr(logits_out), ids.data_ptr(), gp.data_ptr(), lr.data_ptr(),
                          tc.data_ptr(), st)
        else:
            logits = ws["logits"] if logits_out is None else logits_out
            if self.wide_gate:
                _grouped_gemm(torch.float32, x.float(), S, M, self.wg32, E, None, logits, 1, None,
                              0, None, S, S, _lib.MOE_ACT_NONE)
            else:
                _grouped_gemm(self.dtype, x, S, M, self.wg, E, None, logits, 1, None, 0, None, S,
                              S, _lib.MOE_ACT_NONE)
            probs = None
            if aux:
                probs = ws.setdefault("probs", torch.empty((S, E), dtype=torch.float32,
                                                           device=self.device))
            _lib.call("moe_topk_gate", logits.data_ptr(), _lib.MOE_F32, S, E, k, ids.data_ptr(),
                      gp.data_ptr(), _lib.ptr(probs), st)
            _lib.call("moe_plan_tiles", ids.data_ptr(), S, E, k, lr.data_ptr(), tc.data_ptr(), st)
        ph("scan")
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, cap, None, ws["tile_offsets"].data_ptr(),
                  ws["totals"].data_ptr(), ws["load"].data_ptr(), st)
        if aux:
            if self.dtype == torch.bfloat16 and not self.wide_gate:
                _lib.call("moe_load_balance_loss_from_stats", ws["totals"].data_ptr(),
                          ws["probsum"].data_ptr(), S, E, k, ws["aux"].data_ptr(), st)
            else:
                lib = _lib.load()
                wsb = lib.moe_load_balance_workspace_bytes(E)
                scratch = ws.setdefault("aux_ws", torch.empty(wsb // 8, dtype=torch.float64,
                                                              device=self.device))
                _lib.call("moe_load_balance_loss", ids.data_ptr(), S, E, k, ws["probs"].data_ptr(),
                          _lib.MOE_F32, ws["aux"].data_ptr(), scratch.data_ptr(), wsb, st)
            self.last_aux_loss = ws["aux"]
        ph("dispatch")
        if self.fused_combine:
            _lib.call("moe_dispatch_fused", x.data_ptr(), S, M * x.element_size(), E, k, cap,
                      ids.data_ptr(), lr.data_ptr(), ws["tile_offsets"].data_ptr(), gp.data_ptr(),
                      ws["slots"].data_ptr(), _lib.ptr(ws["xbuf"]), ws["row_token"].data_ptr(),
                      ws["row_prob"].data_ptr(), out.data_ptr(), st)
            if cap > 0:
                ph("gemm1")
                if self.gather_rows:  # A rows = x[row_token[row]] (TMA gather4)
                    _lib.call("moe_grouped_gemm_bf16_gather", x.data_ptr(), S,
                              ws["row_token"].data_ptr(), M, self.w1.data_ptr(), E * F, F,
                              self.b1.data_ptr(), ws["h"].data_ptr(), E, cap, ws["load"].data_ptr(),
                              0, cap, _lib.MOE_ACT_GELU | _lib.MOE_GEMM_PAD_SCRATCH, st)
                else:
                    _grouped_gemm(self.dtype, ws["xbuf"], E * cap, M, self.w1, F, self.b1, ws["h"],
                                  E, None, cap, ws["load"], 0, cap, _lib.MOE_ACT_GELU,
                                  scratch_pad=True)
                ph("gemm2")  # + combine + residual in the epilogue
                _lib.call("moe_grouped_gemm_bf16_combine", ws["h"].data_ptr(), E * cap, F,
                          self.w2.data_ptr(), E * M, M, self.b2.data_ptr(), E, None, cap,
                          ws["load"].data_ptr(), 0, None, cap, ws["row_token"].data_ptr(),
                          ws["row_prob"].data_ptr(), x.data_ptr(), out.data_ptr(), None, st)
            ph(None)
            return out
        _lib.call("moe_dispatch", x.data_ptr(), S, M * x.element_size(), E, k, cap, ids.data_ptr(),
                  lr.data_ptr(), ws["tile_offsets"].data_ptr(), ws["slots"].data_ptr(),
                  ws["xbuf"].data_ptr(), st)
        if ws["grouped_shared"]:
            G = ws["G"]
            ph("gemm1")  # experts + shared MLP (x rows) in one launch, bias + GELU
            _lib.call("moe_residual_gemm_bf16", ws["xbuf"].data_ptr(), E * cap, x.data_ptr(), S, E,
                      M, self.w1_all.data_ptr(), (E + 1) * F, F, self.b1_all.data_ptr(),
                      ws["h"].data_ptr(), G, cap, ws["rows_all"].data_ptr(),
                      ws["widx"].data_ptr(), cap, 1, 0, None, None, None, k, cap, None, None, S,
                      None, st)
            ph("gemm2")  # experts -> y; shared groups: (x + sum p*y) + shared MLP -> out
            _lib.call("moe_residual_gemm_bf16", ws["h"].data_ptr(), G * cap, None, 0, 0, F,
                      self.w2_all.data_ptr(), (E + 1) * M, M, self.b2_all.data_ptr(),
                      ws["y"].data_ptr(), G, cap, ws["rows_all"].data_ptr(),
                      ws["widx"].data_ptr(), cap, 0, E, ids.data_ptr(), ws["slots"].data_ptr(),
                      gp.data_ptr(), k, cap, x.data_ptr(), out.data_ptr(), S, None, st)
            ph(None)
            return out
        if cap > 0:
            ph("gemm1")
            _grouped_gemm(self.dtype, ws["xbuf"], E * cap, M, self.w1, F, self.b1, ws["h"], E,
                          None, cap, ws["load"], 0, cap, _lib.MOE_ACT_GELU, scratch_pad=True)
            ph("gemm2")
            _grouped_gemm(self.dtype, ws["h"], E * cap, F, self.w2, M, self.b2, ws["y"], E, None,
                          cap, ws["load"], 0, cap, _lib.MOE_ACT_NONE, scratch_pad=True)
        shared_out = None
        if self.shared is not None and self.dtype == torch.bfloat16:
            # Residual-MoE, shared MLP not grouped (small capacity): shared GEMM1, then
            # its GEMM2 with the combine + both residual adds in the epilogue, the same
            # arithmetic as the grouped launch (arch.py:389-391)
            ph("shared_mlp")
            sh = self.shared
            _grouped_gemm(self.dtype, x, S, M, sh.w1, F, sh.b1, ws["hs"], 1, None, 0, None, S, S,
                          _lib.MOE_ACT_GELU, scratch_pad=True)
            _lib.call("moe_residual_gemm_bf16", ws["hs"].data_ptr(), S, None, 0, 0, F,
                      sh.w2.data_ptr(), M, M, sh.b2.data_ptr(), ws["y"].data_ptr(), 1, S,
                      ws["sh_rows"].data_ptr(), ws["sh_w"].data_ptr(), S, 0, 0, ids.data_ptr(),
                      ws["slots"].data_ptr(), gp.data_ptr(), k, cap, x.data_ptr(),
                      out.data_ptr(), S, None, st)
            ph(None)
            return out
        if self.shared is not None:
            ph("shared_mlp")
            shared_out = self.shared(x, ws["hs"], ws["ys"])
        ph("combine")
        _lib.call("moe_combine", ws["y"].data_ptr(), _lib.dtype_code(self.dtype), S, M, E, k, cap,
                  ids.data_ptr(), ws["slots"].data_ptr(), None, gp.data_ptr(), _lib.MOE_F32,
                  x.data_ptr(), _lib.ptr(shared_out), out.data_ptr(), 1, st)
        ph(None)
        return out

    def forward_train(self, x: torch.Tensor) -> torch.Tensor:
        """Forward keeping the backward context (bf16; ``train.forward_train``)."""
        from .train import forward_train

        return forward_train(self, x)

    def backward(self, dout: torch.Tensor) -> dict:
        """Gradients of sum(out * dout) w.r.t. x and every parameter for the last
        ``forward_train`` (``train.backward``), in the reference layouts."""
        from .train import backward

        self.grads = backward(self, dout)
        return self.grads

    def graphed(self, S: int):
        """This layer's forward for batches of S tokens as one CUDA graph
        (``pipeline.GraphedForward``)."""
        from .pipeline import GraphedForward

        return GraphedForward(self, S, self.M, self.dtype, self.device)

    def kept_assignments(self, S: int) -> int:
        """Kept (non-dropped) assignments of the last forward of size S (host sync)."""
        return int(self._ws[S]["load"].sum().item())

    def plan(self, S: int):
        """(ids, gate_probs, slots, expert_load, capacity) of the last forward of size S."""
        ws = self._ws[S]
        return ws["ids"], ws["gp"], ws["slots"], ws["load"], ws["cap"]


# ---------------------------------------------------------------------------
# reference-shaped entry points
# ---------------------------------------------------------------------------


def load_balance_loss(plan, probs) -> float:
    """E * sum_e (assignment fraction_e) * (mean gate prob_e), fractions taken
    before capacity drops (arch.py:297-313), computed on the device in float64."""
    from .gating import _dev, _is_torch

    as_np = not _is_torch(probs)
    p = np.asarray(probs, dtype=np.float64) if as_np else probs
    e = plan.num_experts
    if len(p.shape) != 2 or tuple(p.shape) != (plan.num_tokens, e):
        raise ShapeError(f"probs shape {tuple(p.shape)} does not match plan")
    if plan.num_tokens == 0:
        return 0.0
    pd = _dev(p)
    if pd.dtype not in (torch.float32, torch.float64):
        pd = pd.float()
    raw = plan.expert_ids
    if (bool(((raw < 0) | (raw >= e)).any()) if _is_torch(raw) else
            bool(np.any((np.asarray(raw) < 0) | (np.asarray(raw) >= e)))):
        # np.bincount rejects negative ids and longer counts do not broadcast
        # against the E mean probabilities (arch.py:310-313)
        raise ValueError(f"expert ids must lie in [0, {e})")
    ids = _dev(np.asarray(raw, dtype=np.int32) if not _is_torch(raw) else raw,
               torch.int32).to(pd.device)
    lib = _lib.load()
    wsb = lib.moe_load_balance_workspace_bytes(e)
    ws = torch.empty(wsb // 8, dtype=torch.float64, device=pd.device)
    out = torch.empty(1, dtype=torch.float64, device=pd.device)
    _lib.call("moe_load_balance_loss", ids.data_ptr(), plan.num_tokens, e, plan.k, pd.data_ptr(),
              _lib.dtype_code(pd.dtype), out.data_ptr(), ws.data_ptr(), wsb, _lib.stream_ptr())
    return float(out.item())


def _input(x):
    """-> (device tensor, how to return). NumPy/Tensor inputs run the fp32 path."""
    raw = as_array(x)
    if isinstance(raw, torch.Tensor):
        dev = _lib.require_device(raw)
        t = raw.to(dev)
        if t.dtype not in (torch.bfloat16, torch.float32):
            t = t.float()
        return t, "torch"
    arr = np.asarray(raw, dtype=np.float64)
    if arr.ndim != 2:
        raise ShapeError(f"batch must be 2-D, got shape {arr.shape}")
    dev = _lib.require_device(None)
    kind = "tensor" if hasattr(x, "value") else "numpy"
    return torch.as_tensor(arr, device=dev).float(), kind


def _output(t: torch.Tensor, kind: str):
    if kind == "torch":
        return t
    arr = t.detach().float().cpu().numpy().astype(np.float64)
    return Tensor(arr) if kind == "tensor" else arr


def forward_ffn(x, p: FfnParams):
    """gelu(x @ w1 + b1) @ w2 + b2 (arch.py:368-369) on the device."""
    t, kind = _input(x)
    m = t.shape[1]
    if isinstance(p, DenseFfn):
        ffn = p
    else:
        w1 = as_array(p.w1)
        ffn = DenseFfn(p, int(w1.shape[0]), t.dtype, t.device)
    if m != ffn.M:
        raise ShapeError(f"batch width {m} does not match ffn width {ffn.M}")
    return _output(ffn(t.to(ffn.dtype).contiguous()), kind)


def forward_layer(x, spec: LayerSpec, params):
    """One block's feed-forward slot with its residual skip (arch.py:372-392).

    ``params``: a ``MoeLayer`` (pre-packed, the fast path), reference-style
    ``MoeLayerParams`` for a moe spec, or ``FfnParams`` for a dense spec.
    NumPy / Tensor inputs run the fp32 path and come back as float64."""
    t, kind = _input(x)
    if t.shape[1] != spec.hidden:
        raise ShapeError(f"batch width {t.shape[1]} does not match layer hidden {spec.hidden}")
    if spec.kind == "dense":
        ffn = params if isinstance(params, DenseFfn) else DenseFfn(params, spec.hidden, t.dtype,
                                                                  t.device)
        xt = t.to(ffn.dtype).contiguous()
        y = ffn(xt)
        out = torch.empty_like(xt)
        s = xt.shape[0]
        if s:
            # out = x + ffn(x): the combine kernel with no routed rows (k=1, all dropped)
            ids = torch.zeros((s, 1), dtype=torch.int32, device=t.device)
            slots = torch.full((s, 1), -1, dtype=torch.int32, device=t.device)
            gp = torch.zeros((s, 1), dtype=torch.float32, device=t.device)
            _lib.call("moe_combine", None, _lib.dtype_code(xt.dtype), s, spec.hidden, 1, 1, 0,
                      ids.data_ptr(), slots.data_ptr(), None, gp.data_ptr(), _lib.MOE_F32,
                      xt.data_ptr(), y.data_ptr(), out.data_ptr(), 1, _lib.stream_ptr())
        return _output(out, kind)
    layer = params if isinstance(params, MoeLayer) else MoeLayer(spec, params, t.dtype, t.device)
    return _output(layer(t), kind)
