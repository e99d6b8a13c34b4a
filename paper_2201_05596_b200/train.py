"""Training support for ``MoeLayer`` (bf16): a forward that keeps what the
backward needs, and the backward itself.

Reference semantics (arch.py:372-413 on the tensor.py tape): the output is
x + sum over kept (t, e) of p_te * FFN_e(x_t) [+ shared MLP(x)], with
p = row_softmax(x @ W_g) at the chosen experts; gradients flow through p (and
so into W_g and x), through each expert FFN, and through the residual skip;
routing decisions (top-k, capacity slots) are constants.

Device plan (every step a libmoe_b200 kernel; GEMMs on tcgen05):

  forward   gate GEMM (logits kept) -> scan -> dispatch -> GEMM1 + GELU,
            saving the pre-activation a -> GEMM2 -> y kept -> combine
  backward  dY = p*dOut and dp = <dOut, y>            (moe_combine_bwd_bf16)
            dA = (dY @ W2^T) * gelu'(a)               (grouped GEMM, GELU_BWD epilogue)
            dXr = dA @ W1^T                           (grouped GEMM)
            dW2 = h^T dY, dW1 = x_e^T dA, db          (per-expert transposes + grouped GEMMs)
            dlogits = s * (g - <g, s>)                (moe_gate_bwd)
            dW_g = x^T dlogits, dx_gate = dlogits W_g^T
            shared MLP: the same with one group of all S rows
            dx = dOut + scatter(dXr) + dx_gate + dx_shared  (moe_bwd_dx_bf16)
"""

from __future__ import annotations

import torch

from . import _lib


def _gemm(a, a_rows, K, w, N, bias, d, G, row_stride, rows, rows_const, max_rows, act=0,
          aux=None):
    """act may carry MOE_GEMM_PAD_SCRATCH: the groups' padding rows of d are never
    read (combine / dx assembly read kept slots only), so the GEMM may use its
    TMA-store epilogue and 256x512 tiles."""
    st = _lib.stream_ptr()
    if act in (_lib.MOE_ACT_GELU_SAVE, _lib.MOE_ACT_GELU_BWD):
        _lib.call("moe_grouped_gemm_bf16_aux", a.data_ptr(), a_rows, K, w.data_ptr(), w.shape[0],
                  N, _lib.ptr(bias), d.data_ptr(), G, None, row_stride, _lib.ptr(rows),
                  rows_const, None, max_rows, act, aux.data_ptr(), st)
    else:
        _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), a_rows, K, w.data_ptr(), w.shape[0], N,
                  _lib.ptr(bias), d.data_ptr(), G, None, row_stride, _lib.ptr(rows), rows_const,
                  None, max_rows, act, st)


def _wgrad(x, P, y, Q, G, k_stride, k_rows, k_rows_const):
    """bf16 (G, P, Q): X_g^T Y_g over each group's first k_rows[g] rows (no transposes)."""
    out = torch.empty((G, P, Q), dtype=torch.bfloat16, device=x.device)
    _lib.call("moe_grouped_gemm_bf16_wgrad", x.data_ptr(), x.shape[0], P, y.data_ptr(), Q, G,
              k_stride, _lib.ptr(k_rows), k_rows_const, out.data_ptr(), _lib.stream_ptr())
    return out


def _colsum(x, W, G, row_stride, rows, rows_const):
    out = torch.zeros((G, W), dtype=torch.float32, device=x.device)
    _lib.call("moe_colsum_rows_bf16", x.data_ptr(), W, G, row_stride, _lib.ptr(rows), rows_const,
              out.data_ptr(), _lib.stream_ptr())
    return out


def _orig_weights(layer):
    """Reference-layout copies of the weights for the data-gradient GEMMs:
    W1 (E*M, F), W2 (E*F, M), [W_g | W_g] (M, 2*Epad) (made once, on first backward)."""
    if getattr(layer, "_w_orig", None) is None:
        E, M, F = layer.E, layer.M, layer.F
        w1o = layer.w1.view(E, F, M).transpose(1, 2).contiguous().view(E * M, F)
        w2o = layer.w2.view(E, M, F).transpose(1, 2).contiguous().view(E * F, M)
        wgo = layer.wg.t().contiguous()  # (M, Epad), zero beyond E
        wgo = torch.cat([wgo, wgo], dim=1).contiguous()  # (M, 2*Epad): [Wg | Wg] for hi/lo dlogits
        sh = None
        if layer.shared is not None:
            s = layer.shared
            sh = (s.w1.t().contiguous(), s.w2.t().contiguous())  # (M, F), (F, M)
        layer._w_orig = (w1o, w2o, wgo, sh)
    return layer._w_orig


def forward_train(layer, x: torch.Tensor) -> torch.Tensor:
    """Forward that saves the backward context (bf16 only)."""
    if layer.dtype != torch.bfloat16:
        raise NotImplementedError("the training path is bf16 (tcgen05)")
    if getattr(layer, "wide_gate", False):
        raise NotImplementedError("the training path covers E <= 256 (the fused tcgen05 gate)")
    x = x.to(device=layer.device, dtype=layer.dtype).contiguous()
    S = x.shape[0]
    ws = layer.workspace(S)
    cap, E, M, F, k = ws["cap"], layer.E, layer.M, layer.F, layer.k
    st = _lib.stream_ptr()
    dev = layer.device
    out = torch.empty_like(x)
    logits = torch.empty((S, E), dtype=torch.float32, device=dev)
    ids, gp, lr, tc = ws["ids"], ws["gp"], ws["local_rank"], ws["tile_counts"]
    a = torch.empty((max(E * cap, 1), F), dtype=torch.bfloat16, device=dev)
    h = torch.empty_like(a)
    xbuf = torch.empty((max(E * cap, 1), M), dtype=torch.bfloat16, device=dev)
    y = torch.empty_like(xbuf)
    slots = torch.empty_like(ids)
    load = torch.empty_like(ws["load"])
    if S:
        _lib.call("moe_gate_gemm_bf16", x.data_ptr(), layer.wg.data_ptr(), S, M, E, k,
                  logits.data_ptr(), ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(),
                  st)
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, cap, None, ws["tile_offsets"].data_ptr(),
                  ws["totals"].data_ptr(), load.data_ptr(), st)
    # k=1 without a shared MLP: combine + residual fused into GEMM2's epilogue, which
    # also keeps y (the gate-probability gradient needs it); otherwise a separate combine
    fused = k == 1 and layer.shared is None
    if S and fused:
        i32 = dict(dtype=torch.int32, device=dev)
        row_token = torch.empty(max(E * cap, 1), **i32)
        row_prob = torch.empty(max(E * cap, 1), dtype=torch.float32, device=dev)
        _lib.call("moe_dispatch_fused", x.data_ptr(), S, M * 2, E, k, cap, ids.data_ptr(),
                  lr.data_ptr(), ws["tile_offsets"].data_ptr(), gp.data_ptr(), slots.data_ptr(),
                  xbuf.data_ptr(), row_token.data_ptr(), row_prob.data_ptr(), out.data_ptr(), st)
        if cap:
            _gemm(xbuf, E * cap, M, layer.w1, F, layer.b1, h, E, cap, load, 0, cap,
                  _lib.MOE_ACT_GELU_SAVE, a)
            _lib.call("moe_grouped_gemm_bf16_combine", h.data_ptr(), E * cap, F,
                      layer.w2.data_ptr(), E * M, M, layer.b2.data_ptr(), E, None, cap,
                      load.data_ptr(), 0, None, cap, row_token.data_ptr(), row_prob.data_ptr(),
                      x.data_ptr(), out.data_ptr(), y.data_ptr(), st)
    elif S:
        _lib.call("moe_dispatch", x.data_ptr(), S, M * 2, E, k, cap, ids.data_ptr(),
                  lr.data_ptr(), ws["tile_offsets"].data_ptr(), slots.data_ptr(),
                  xbuf.data_ptr(), st)
        if cap:
            _gemm(xbuf, E * cap, M, layer.w1, F, layer.b1, h, E, cap, load, 0, cap,
                  _lib.MOE_ACT_GELU_SAVE, a)
            _gemm(h, E * cap, F, layer.w2, M, layer.b2, y, E, cap, load, 0, cap, _lib.MOE_GEMM_PAD_SCRATCH)
    sh_ctx = None
    if layer.shared is not None and S:
        # shared MLP: GEMM1 saving its pre-activation, then GEMM2 with the combine and
        # both residual adds in its epilogue (the inference arithmetic, arch.py:389-391)
        s = layer.shared
        i32 = dict(dtype=torch.int32, device=dev)
        a_s = torch.empty((S, F), dtype=torch.bfloat16, device=dev)
        h_s = torch.empty_like(a_s)
        _gemm(x, S, M, s.w1, F, s.b1, h_s, 1, 0, None, S, S, _lib.MOE_ACT_GELU_SAVE, a_s)
        sh_rows, sh_w = torch.tensor([S], **i32), torch.zeros(1, **i32)  # (kept alive)
        _lib.call("moe_residual_gemm_bf16", h_s.data_ptr(), S, None, 0, 0, F, s.w2.data_ptr(), M,
                  M, s.b2.data_ptr(), y.data_ptr(), 1, S, sh_rows.data_ptr(), sh_w.data_ptr(), S,
                  0, 0, ids.data_ptr(), slots.data_ptr(), gp.data_ptr(), k, cap, x.data_ptr(),
                  out.data_ptr(), S, None, st)
        sh_ctx = (a_s, h_s)
    elif S and not fused:
        _lib.call("moe_combine", y.data_ptr(), _lib.MOE_BF16, S, M, E, k, cap, ids.data_ptr(),
                  slots.data_ptr(), None, gp.data_ptr(), _lib.MOE_F32, x.data_ptr(),
                  None, out.data_ptr(), 1, st)
    layer._train_ctx = dict(x=x, S=S, cap=cap, logits=logits, ids=ids.clone(), gp=gp.clone(),
                            slots=slots, load=load, xbuf=xbuf, a=a, h=h, y=y, shared=sh_ctx)
    return out


def backward(layer, dout: torch.Tensor) -> dict:
    """Gradients of sum(out * dout) for the last ``forward_train``.

    Returns {"x", "gate_w" (M, E), "w1" (E, M, F), "b1" (E, F), "w2" (E, F, M),
    "b2" (E, M)} plus "shared" = {"w1", "b1", "w2", "b2"} for Residual-MoE;
    weight gradients in the reference layouts (arch.py:321-344)."""
    c = layer._train_ctx
    x, S, cap = c["x"], c["S"], c["cap"]
    E, M, F, k = layer.E, layer.M, layer.F, layer.k
    dev = layer.device
    st = _lib.stream_ptr()
    dout = dout.to(device=dev, dtype=torch.bfloat16).contiguous()
    w1o, w2o, wgo, sh_o = _orig_weights(layer)
    ids, gp, slots, load = c["ids"], c["gp"], c["slots"], c["load"]
    f32 = dict(dtype=torch.float32, device=dev)
    grads = {}
    dp = torch.zeros((S, k), **f32)
    dxr = None
    if cap and S:
        dy = torch.empty((E * cap, M), dtype=torch.bfloat16, device=dev)
        _lib.call("moe_combine_bwd_bf16", dout.data_ptr(), c["y"].data_ptr(), S, M, E, k, cap,
                  ids.data_ptr(), slots.data_ptr(), gp.data_ptr(), dy.data_ptr(), dp.data_ptr(),
                  st)
        dA = torch.empty((E * cap, F), dtype=torch.bfloat16, device=dev)
        _gemm(dy, E * cap, M, w2o, F, None, dA, E, cap, load, 0, cap, _lib.MOE_ACT_GELU_BWD,
              c["a"])
        dxr = torch.empty((E * cap, M), dtype=torch.bfloat16, device=dev)
        _gemm(dA, E * cap, F, w1o, M, None, dxr, E, cap, load, 0, cap, _lib.MOE_GEMM_PAD_SCRATCH)
        # weight gradients: contract over each expert's kept rows, read MN-major
        # straight from the saved activations
        db2 = _colsum(dy, M, E, cap, load, 0)
        db1 = _colsum(dA, F, E, cap, load, 0)
        dw2 = _wgrad(c["h"], F, dy, M, E, cap, load, 0)
        dw1 = _wgrad(c["xbuf"], M, dA, F, E, cap, load, 0)
        grads.update(w1=dw1, b1=db1, w2=dw2, b2=db2)
    else:
        grads.update(w1=torch.zeros((E, M, F), dtype=torch.bfloat16, device=dev),
                     b1=torch.zeros((E, F), **f32),
                     w2=torch.zeros((E, F, M), dtype=torch.bfloat16, device=dev),
                     b2=torch.zeros((E, M), **f32))
    # gate: through row_softmax into W_g and x
    epad = layer.epad
    # dlogits as bf16 hi|lo pairs (S, 2*Epad): dx's gate term = [hi|lo] @ [Wg|Wg]^T
    dlog = torch.empty((max(S, 1), 2 * epad), dtype=torch.bfloat16, device=dev)
    dxg = torch.empty((S, M), dtype=torch.bfloat16, device=dev)
    dwg = torch.zeros((M, 2 * epad), **f32)
    if S:
        _lib.call("moe_gate_bwd", c["logits"].data_ptr(), S, E, epad, k, ids.data_ptr(),
                  slots.data_ptr(), dp.data_ptr(), dlog.data_ptr(), 1, st)
        _gemm(dlog, S, 2 * epad, wgo, M, None, dxg, 1, 0, None, S, S, _lib.MOE_GEMM_PAD_SCRATCH)
        _lib.call("moe_gemm_bf16_wgrad_f32", x.data_ptr(), S, M, dlog.data_ptr(), 2 * epad,
                  dwg.data_ptr(), st)
    grads["gate_w"] = dwg[:, :E] + dwg[:, epad:epad + E]  # hi + lo (fp32)
    # shared MLP (Residual-MoE)
    dxs = None
    if layer.shared is not None and S:
        a_s, h_s = c["shared"]
        s1o, s2o = sh_o
        dA_s = torch.empty((S, F), dtype=torch.bfloat16, device=dev)
        _gemm(dout, S, M, s2o, F, None, dA_s, 1, 0, None, S, S, _lib.MOE_ACT_GELU_BWD, a_s)
        dxs = torch.empty((S, M), dtype=torch.bfloat16, device=dev)
        _gemm(dA_s, S, F, s1o, M, None, dxs, 1, 0, None, S, S, _lib.MOE_GEMM_PAD_SCRATCH)
        sdb2 = _colsum(dout, M, 1, 0, None, S)
        sdb1 = _colsum(dA_s, F, 1, 0, None, S)
        sdw2 = _wgrad(h_s, F, dout, M, 1, 0, None, S)[0]
        sdw1 = _wgrad(x, M, dA_s, F, 1, 0, None, S)[0]
        grads["shared"] = dict(w1=sdw1, b1=sdb1, w2=sdw2, b2=sdb2)
    dx = torch.empty_like(dout)
    if S:
        _lib.call("moe_bwd_dx_bf16", dout.data_ptr(), _lib.ptr(dxr), S, M, E, k, cap,
                  ids.data_ptr(), slots.data_ptr(), dxg.data_ptr(), _lib.ptr(dxs), dx.data_ptr(),
                  st)
    grads["x"] = dx
    return grads


class MoeFunction(torch.autograd.Function):
    """torch.autograd binding: y = MoeFunction.apply(x, layer) participates in a
    PyTorch graph; x.grad comes back and the parameter gradients are left on
    ``layer.grads`` after backward."""

    @staticmethod
    def forward(ctx, x, layer):
        ctx.layer = layer
        return forward_train(layer, x)

    @staticmethod
    def backward(ctx, dout):
        g = backward(ctx.layer, dout)
        ctx.layer.grads = g
        return g["x"], None
