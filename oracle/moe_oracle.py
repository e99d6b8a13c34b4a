"""CPU oracle for the DeepSpeed-MoE layer forward (TEST INFRASTRUCTURE ONLY).

This module is the parity checker for the B200 path. It is a float64 NumPy
restatement of the reference package ``moekit`` (``/root/reference/pkg``),
function by function, each citing the reference ``file:line`` it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg (and ``bench.py --impl reference``) may import it.
The product package ``paper_2201_05596_b200`` never imports this module and
has no CPU fallback.

Parity pinning: every function here is checked against golden vectors that
were produced by importing the reference itself (``tests/golden/make_golden.py``
writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks them).
The routing functions are bit-exact against those vectors; the layer forward
matches the reference to <= 1e-12 (both are float64 NumPy with the same
operation order, in practice bitwise equal).

Algorithm sources (third-party): all arithmetic is NumPy (>=1.24 unpinned in
``pkg/pyproject.toml:10``; 2.3.5 in this image) with OpenBLAS dgemm for
``@``. Nothing is vendored in the reference.
"""

from __future__ import annotations

import math

import numpy as np

DROPPED = -1  # gating.py:52


# ---------------------------------------------------------------------------
# gating
# ---------------------------------------------------------------------------


def capacity(num_experts: int, k: int, capacity_factor: float, num_tokens: int) -> int:
    """Slots per expert: ceil(cf * S * k / E) evaluated in float64, left to
    right, and 0 for an empty batch (gating.py:77-80)."""
    if num_tokens == 0:
        return 0
    return int(np.ceil(capacity_factor * num_tokens * k / num_experts))


def softmax_rows(logits: np.ndarray) -> np.ndarray:
    """Max-shifted row softmax (gating.py:156-158, tensor.py:248-251)."""
    if logits.size == 0:
        return logits.copy()
    z = logits - logits.max(axis=1, keepdims=True)
    ez = np.exp(z)
    return ez / ez.sum(axis=1, keepdims=True)


def top_k_gate(logits: np.ndarray, num_experts: int, k: int):
    """Top-k expert choice per token (gating.py:142-163).

    Returns (expert_ids (S,k) int64, gate_probs (S,k) f64, probs (S,E) f64).
    Order is descending logit with ties to the lower expert index (a stable
    sort of the negated logits, gating.py:159-161); probabilities are the
    full-E softmax gathered at the chosen ids, not renormalised
    (gating.py:145-147, :162).
    """
    logits = np.asarray(logits, dtype=np.float64)
    assert logits.ndim == 2 and logits.shape[1] == num_experts
    probs = softmax_rows(logits)
    ids = np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int64)
    if logits.size:
        gp = np.take_along_axis(probs, ids, axis=1)
    else:
        gp = np.zeros(ids.shape, dtype=np.float64)
    return ids, gp, probs


def exclusive_scan_blelloch(values: np.ndarray) -> np.ndarray:
    """Work-efficient exclusive prefix sum over a power-of-two padded buffer
    (gating.py:171-203). Integer/bool input -> int64 (exact); float input ->
    float64 summed in the up-sweep/down-sweep tree order."""
    v = np.asarray(values)
    assert v.ndim == 1
    n = v.shape[0]
    is_int = v.dtype.kind in "iub"
    out_dtype = np.int64 if is_int else np.float64
    if n == 0:
        return np.zeros(0, dtype=out_dtype if is_int else v.dtype)
    size = 1 << (n - 1).bit_length()
    tree = np.zeros(size, dtype=out_dtype)
    tree[:n] = v
    stride = 1
    while stride < size:  # up-sweep: right child of each pair absorbs the left
        tree[2 * stride - 1 :: 2 * stride] += tree[stride - 1 :: 2 * stride]
        stride <<= 1
    tree[size - 1] = 0
    stride = size >> 1
    while stride:  # down-sweep: left gets parent, right gets parent + old left
        left = tree[stride - 1 :: 2 * stride].copy()
        tree[stride - 1 :: 2 * stride] = tree[2 * stride - 1 :: 2 * stride]
        tree[2 * stride - 1 :: 2 * stride] += left
        stride >>= 1
    return tree[:n]


def build_dispatch_plan(expert_ids: np.ndarray, num_experts: int, k: int,
                        capacity_factor: float):
    """Capacity slots in flattened token-major order (gating.py:211-247).

    For each expert, an assignment's slot is the exclusive running count of
    earlier assignments to that expert (the Blelloch scan of the expert's
    indicator, gating.py:229-234); slot >= capacity -> DROPPED
    (gating.py:235-236); expert_load counts kept assignments (gating.py:237).
    Returns (slots (S,k) int64, expert_load (E,) int64, capacity).
    """
    ids = np.asarray(expert_ids, dtype=np.int64)
    s = ids.shape[0]
    cap = capacity(num_experts, k, capacity_factor, s)
    flat = ids.reshape(-1)
    slots = np.full(flat.shape[0], DROPPED, dtype=np.int64)
    load = np.zeros(num_experts, dtype=np.int64)
    for e in range(num_experts):
        hit = flat == e
        before = exclusive_scan_blelloch(hit.astype(np.int64))
        pos = np.flatnonzero(hit)
        slot = before[pos]
        keep = slot < cap
        slots[pos[keep]] = slot[keep]
        load[e] = int(keep.sum())
    return slots.reshape(s, k), load, cap


def build_dispatch_plan_fast(expert_ids: np.ndarray, num_experts: int, k: int,
                             capacity_factor: float):
    """Same result as :func:`build_dispatch_plan` via one stable sort (used
    for the large C3-scale parity checks where E scans of 64K are slow)."""
    ids = np.asarray(expert_ids, dtype=np.int64)
    s = ids.shape[0]
    cap = capacity(num_experts, k, capacity_factor, s)
    flat = ids.reshape(-1)
    order = np.argsort(flat, kind="stable")
    sorted_ids = flat[order]
    counts = np.bincount(flat, minlength=num_experts)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    rank = np.arange(flat.shape[0]) - starts[sorted_ids]
    slot_flat = np.empty(flat.shape[0], dtype=np.int64)
    slot_flat[order] = rank
    slot_flat[slot_flat >= cap] = DROPPED
    load = np.minimum(counts, cap).astype(np.int64)
    return slot_flat.reshape(s, k), load, cap


def scatter_tokens(batch: np.ndarray, expert_ids: np.ndarray, slots: np.ndarray,
                   num_experts: int, cap: int):
    """Table-driven dispatch (gating.py:255-278): data[e, slot] = batch[t] for
    kept assignments, unoccupied slots zero. Returns (data, occupied)."""
    batch = np.asarray(batch, dtype=np.float64)
    m = batch.shape[1]
    data = np.zeros((num_experts, cap, m))
    occupied = np.zeros((num_experts, cap), dtype=bool)
    kept = slots != DROPPED
    tok = np.nonzero(kept)[0]
    e = expert_ids[kept]
    sl = slots[kept]
    data[e, sl] = batch[tok]
    occupied[e, sl] = True
    return data, occupied


def combine_tokens(data: np.ndarray, expert_ids: np.ndarray, slots: np.ndarray,
                   gate_probs: np.ndarray) -> np.ndarray:
    """Table-driven combine (gating.py:281-307): out[t] = sum over kept
    assignments, in token-major order, of gate_prob * data[e, slot]."""
    s = expert_ids.shape[0]
    out = np.zeros((s, data.shape[2]))
    kept = slots != DROPPED
    tok = np.nonzero(kept)[0]
    contrib = gate_probs[kept][:, None] * data[expert_ids[kept], slots[kept]]
    np.add.at(out, tok, contrib)
    return out


def onehot_dispatch_mask(expert_ids: np.ndarray, num_experts: int, cap: int) -> np.ndarray:
    """(S, E, c) one-hot mask from an independent cumsum (gating.py:315-331)."""
    s, k = expert_ids.shape
    flat = expert_ids.reshape(-1)
    hot = flat[:, None] == np.arange(num_experts)[None, :]
    running = np.cumsum(hot, axis=0) - hot
    mask = np.zeros((s * k, num_experts, cap))
    r, c = np.where(hot)
    sl = running[r, c]
    ok = sl < cap
    mask[r[ok], c[ok], sl[ok]] = 1.0
    return mask.reshape(s, k, num_experts, cap).sum(axis=1)


def sparse_dispatch_oracle(batch, expert_ids, num_experts, cap):
    """Literal one-hot einsum dispatch (gating.py:334-348)."""
    mask = onehot_dispatch_mask(expert_ids, num_experts, cap)
    return np.einsum("sec,sm->ecm", mask, np.asarray(batch, dtype=np.float64))


def sparse_combine_oracle(outputs, expert_ids, gate_probs, num_experts, cap):
    """Gate-prob weighted one-hot contraction back to tokens (gating.py:351-377):
    every kept assignment (t, j) contributes p[t, j] * outputs[e, slot]; the
    weight tensor is the dispatch mask with each assignment's ones scaled by
    its gate prob, contracted as einsum("sec,ecm->sm")."""
    expert_ids = np.asarray(expert_ids)
    s, k = expert_ids.shape
    flat = expert_ids.reshape(-1)
    hot = flat[:, None] == np.arange(num_experts)[None, :]
    running = np.cumsum(hot, axis=0) - hot
    wmask = np.zeros((s * k, num_experts, cap))
    r, c = np.where(hot)
    sl = running[r, c]
    ok = sl < cap
    wmask[r[ok], c[ok], sl[ok]] = np.asarray(gate_probs, dtype=np.float64).reshape(-1)[r[ok]]
    w = wmask.reshape(s, k, num_experts, cap).sum(axis=1)
    return np.einsum("sec,ecm->sm", w, np.asarray(outputs, dtype=np.float64))


# ---------------------------------------------------------------------------
# layer
# ---------------------------------------------------------------------------

GELU_C = math.sqrt(2.0 / math.pi)


def gelu(x: np.ndarray) -> np.ndarray:
    """tanh-form GELU (tensor.py:219-226)."""
    inner = GELU_C * (x + 0.044715 * x**3)
    return 0.5 * x * (1.0 + np.tanh(inner))


def forward_ffn(x, w1, b1, w2, b2):
    """gelu(x @ w1 + b1) @ w2 + b2 (arch.py:368-369)."""
    return gelu(x @ w1 + b1) @ w2 + b2


def forward_layer_with_logits(x, logits, experts, shared, num_experts, k, capacity_factor):
    """Layer forward given the gate logits (arch.py:372-413).

    ``experts`` is a list of (w1, b1, w2, b2) float64 arrays, ``shared`` the
    Residual-MoE MLP or None. Routing is decided on the logits
    (arch.py:385-386), the combine weight is row_softmax(logits)[t, e]
    (arch.py:387, :408), experts are visited in ascending index with rows in
    slot order and scatter-added into a zero (S, M) accumulator
    (arch.py:399-410); out = x + acc (:389), then + shared MLP (:390-391).
    """
    x = np.asarray(x, dtype=np.float64)
    logits = np.asarray(logits, dtype=np.float64)
    ids, _, probs = top_k_gate(logits, num_experts, k)
    slots, _, _ = build_dispatch_plan(ids, num_experts, k, capacity_factor)
    acc = np.zeros(x.shape)
    kept = slots != DROPPED
    for e in range(num_experts):
        sel = kept & (ids == e)
        if not sel.any():
            continue
        order = np.argsort(slots[sel], kind="stable")
        tokens = np.nonzero(sel)[0][order]
        y = forward_ffn(x[tokens], *experts[e])
        w = probs[tokens, e][:, None]
        contrib = np.zeros(x.shape)
        np.add.at(contrib, tokens, y * w)
        acc = acc + contrib
    out = x + acc
    if shared is not None:
        out = out + forward_ffn(x, *shared)
    return out


def forward_layer(x, gate_w, experts, shared, num_experts, k, capacity_factor):
    """arch.forward_layer (arch.py:372-392) for a moe LayerSpec."""
    x = np.asarray(x, dtype=np.float64)
    logits = x @ np.asarray(gate_w, dtype=np.float64)  # arch.py:384
    return forward_layer_with_logits(x, logits, experts, shared, num_experts, k,
                                     capacity_factor)


def forward_layer_sampled(x, logits, experts, shared, num_experts, k, capacity_factor,
                          expert_subset):
    """Reference output restricted to tokens whose kept assignments all land
    in ``expert_subset`` (plus every fully dropped token): the C3-scale check
    evaluates only a few experts' FFNs. Returns (token_index, out_rows)."""
    x = np.asarray(x, dtype=np.float64)
    logits = np.asarray(logits, dtype=np.float64)
    ids, _, probs = top_k_gate(logits, num_experts, k)
    slots, _, _ = build_dispatch_plan_fast(ids, num_experts, k, capacity_factor)
    kept = slots != DROPPED
    subset = np.zeros(num_experts, dtype=bool)
    subset[list(expert_subset)] = True
    ok = np.all(~kept | subset[ids], axis=1)
    tokens = np.nonzero(ok)[0]
    acc = np.zeros((tokens.shape[0], x.shape[1]))
    for e in sorted(expert_subset):
        for j in range(k):
            sel = kept[tokens, j] & (ids[tokens, j] == e)
            if not sel.any():
                continue
            rows = tokens[sel]
            y = forward_ffn(x[rows], *experts[e])
            acc[sel] += y * probs[rows, e][:, None]
    out = x[tokens] + acc
    if shared is not None:
        out = out + forward_ffn(x[tokens], *shared)
    return tokens, out


def load_balance_loss(expert_ids, probs, num_experts, k):
    """E * sum_e f_e * P_e with pre-drop fractions (arch.py:297-313)."""
    s = expert_ids.shape[0]
    if s == 0:
        return 0.0
    counts = np.bincount(expert_ids.reshape(-1), minlength=num_experts)
    frac = counts / (s * k)
    return float(num_experts * np.sum(frac * probs.mean(axis=0)))


def init_layer_params(hidden, num_experts, residual, rng, scale=0.1):
    """arch.init_layer_params draw order (arch.py:347-365): gate_w (M,E), then
    per expert w1 (M,4M), w2 (4M,M) with zero biases, then the shared MLP."""
    inner = 4 * hidden

    def ffn():
        w1 = rng.standard_normal((hidden, inner)) * scale
        w2 = rng.standard_normal((inner, hidden)) * scale
        return (w1, np.zeros((1, inner)), w2, np.zeros((1, hidden)))

    gate_w = rng.standard_normal((hidden, num_experts)) * scale
    experts = [ffn() for _ in range(num_experts)]
    shared = ffn() if residual else None
    return gate_w, experts, shared


def gelu_grad(x):
    """d gelu / dx, the vjp of tensor.py:229-233."""
    th = np.tanh(GELU_C * (x + 0.044715 * x**3))
    return 0.5 * (1.0 + th) + 0.5 * x * (1.0 - th**2) * GELU_C * (1.0 + 3 * 0.044715 * x**2)


def forward_layer_backward(x, logits, gate_w, experts, shared, num_experts, k, capacity_factor,
                           dout):
    """Gradients of sum(forward_layer(x) * dout), the reference tape's semantics
    (arch.py:372-413 recorded on tensor.py's GradTape): routing is constant;
    the gate gradient flows through row_softmax (tensor.py:263-266) at the
    kept (token, expert) pairs (take_elems vjp, :286-290); experts through
    forward_ffn's matmul/add/gelu vjps; the skip and shared MLP add directly.
    Returns dict(x, gate_w, w1, b1, w2, b2 (lists per expert), shared)."""
    x = np.asarray(x, dtype=np.float64)
    dout = np.asarray(dout, dtype=np.float64)
    ids, _, probs = top_k_gate(logits, num_experts, k)
    slots, _, _ = build_dispatch_plan_fast(ids, num_experts, k, capacity_factor)
    kept = slots != DROPPED
    dx = dout.copy()
    dprobs = np.zeros_like(probs)
    out = dict(w1=[], b1=[], w2=[], b2=[])
    for e in range(num_experts):
        w1, b1, w2, b2 = experts[e]
        sel = kept & (ids == e)
        order = np.argsort(slots[sel], kind="stable")
        tokens = np.nonzero(sel)[0][order]
        if tokens.size == 0:
            out["w1"].append(np.zeros_like(w1)); out["b1"].append(np.zeros_like(b1))
            out["w2"].append(np.zeros_like(w2)); out["b2"].append(np.zeros_like(b2))
            continue
        rows = x[tokens]
        a1 = rows @ w1 + b1
        h = gelu(a1)
        y = h @ w2 + b2
        g = dout[tokens]
        p = probs[tokens, e][:, None]
        dprobs[tokens, e] += (g * y).sum(axis=1)
        dy = g * p
        out["w2"].append(h.T @ dy); out["b2"].append(dy.sum(axis=0, keepdims=True))
        da = (dy @ w2.T) * gelu_grad(a1)
        out["w1"].append(rows.T @ da); out["b1"].append(da.sum(axis=0, keepdims=True))
        np.add.at(dx, tokens, da @ w1.T)
    dlogits = probs * (dprobs - (dprobs * probs).sum(axis=1, keepdims=True))
    out["gate_w"] = x.T @ dlogits
    dx += dlogits @ np.asarray(gate_w, dtype=np.float64).T
    if shared is not None:
        w1, b1, w2, b2 = shared
        a1 = x @ w1 + b1
        h = gelu(a1)
        da = (dout @ w2.T) * gelu_grad(a1)
        out["shared"] = dict(w1=x.T @ da, b1=da.sum(axis=0, keepdims=True), w2=h.T @ dout,
                             b2=dout.sum(axis=0, keepdims=True))
        dx += da @ w1.T
    out["x"] = dx
    return out
