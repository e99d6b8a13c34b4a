"""Numerics of the grouped GEMM kernels against a plain PyTorch reference
(fp32 / fp64 math on the same bf16- or fp32-rounded operands)."""

import pytest
import torch

from paper_2201_05596_b200 import _lib

pytestmark = pytest.mark.gpu


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def _ref(a, w_t, bias, rows, starts, widx, act, N):
    """fp32 reference: for group g, D[rows] = act(A[rows] @ W_w^T + b_w)."""
    out = {}
    for g, (r, s) in enumerate(zip(rows, starts)):
        if r == 0:
            continue
        wi = widx[g]
        w = w_t[wi * N:(wi + 1) * N].float()
        y = a[s:s + r].float() @ w.t()
        if bias is not None:
            y = y + bias[wi]
        out[g] = _gelu(y) if act else y
    return out


@pytest.mark.parametrize("pad", [False, True])
@pytest.mark.parametrize("K,N,act", [(1024, 4096, 1), (4096, 1024, 0), (2048, 8192, 1),
                                     (64, 256, 0), (16, 64, 1), (136, 200, 0), (2048, 96, 1)])
def test_grouped_gemm_bf16(K, N, act, pad):
    torch.manual_seed(K + N)
    G, cap = 5, 300
    rows = [300, 0, 129, 1, 257]
    starts = [g * cap for g in range(G)]
    a = (torch.randn(G * cap, K, device="cuda") * 0.5).to(torch.bfloat16)
    w_t = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(G, N, device="cuda") * 0.1
    d = torch.full((G * cap, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    rows_t = torch.tensor(rows, dtype=torch.int32, device="cuda")
    _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), G * cap, K, w_t.data_ptr(), G * N, N,
              bias.data_ptr(), d.data_ptr(), G, None, cap, rows_t.data_ptr(), 0, None, cap,
              act | (_lib.MOE_GEMM_PAD_SCRATCH if pad else 0), _lib.stream_ptr())
    torch.cuda.synchronize()
    ref = _ref(a, w_t, bias, rows, starts, list(range(G)), act, N)
    for g, want in ref.items():
        got = d[starts[g]:starts[g] + rows[g]].float()
        scale = want.abs().mean().item() + 1e-6
        err = (got - want).abs().max().item()
        assert err <= 2e-2 * (want.abs().max().item() + scale), (g, err)
    if not pad:  # rows beyond each group's count are untouched
        assert torch.isnan(d[cap:2 * cap].float()).all()
        assert torch.isnan(d[2 * cap + 129:3 * cap].float()).all()


@pytest.mark.parametrize("K,N", [(1024, 2048), (512, 1024), (136, 200)])
def test_grouped_gemm_bf16_combine_keeps_y_in_bounds(K, N):
    """Fused-combine GEMM2 of the training forward (train.py:119-122): out[token] =
    x[token] + p * (A W^T + b) for every kept row, y = A W^T + b kept for backward.
    Rows past a group's count are never written, neither in out nor in y - a
    second 256-row tile of group 0 overhangs group 1's block (cap 300)."""
    torch.manual_seed(K + 7 * N)
    G, cap = 5, 300
    rows = [300, 0, 129, 1, 257]
    S = sum(rows)
    a = (torch.randn(G * cap, K, device="cuda") * 0.5).to(torch.bfloat16)
    w_t = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(G, N, device="cuda") * 0.1
    x = torch.randn(S, N, device="cuda").to(torch.bfloat16)
    perm = torch.randperm(S, device="cuda").to(torch.int32)
    row_token = torch.full((G * cap,), -1, dtype=torch.int32, device="cuda")
    row_prob = torch.rand(G * cap, device="cuda")
    n = 0
    for g, r in enumerate(rows):
        row_token[g * cap:g * cap + r] = perm[n:n + r]
        n += r
    out = torch.full((S, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    y = torch.full((G * cap, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    rows_t = torch.tensor(rows, dtype=torch.int32, device="cuda")
    _lib.call("moe_grouped_gemm_bf16_combine", a.data_ptr(), G * cap, K, w_t.data_ptr(), G * N, N,
              bias.data_ptr(), G, None, cap, rows_t.data_ptr(), 0, None, cap,
              row_token.data_ptr(), row_prob.data_ptr(), x.data_ptr(), out.data_ptr(),
              y.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    ref = _ref(a, w_t, bias, rows, [g * cap for g in range(G)], list(range(G)), 0, N)
    for g, want in ref.items():
        sl = slice(g * cap, g * cap + rows[g])
        tol = 2e-2 * (want.abs().max().item() + 1.0)
        assert (y[sl].float() - want).abs().max().item() <= tol, g
        tok = row_token[sl].long()
        want_out = x[tok].float() + row_prob[sl, None] * want
        assert (out[tok].float() - want_out).abs().max().item() <= tol, g
        assert torch.isnan(y[g * cap + rows[g]:(g + 1) * cap].float()).all(), g
    assert torch.isnan(y[cap:2 * cap].float()).all()  # group 1: no rows
    assert not torch.isnan(out.float()).any()  # every token is some kept row


def test_grouped_gemm_bf16_weight_index_and_row_start():
    torch.manual_seed(0)
    K, N = 512, 512
    rows = [200, 64, 333]
    starts = [17, 500, 700]
    widx = [2, 0, 2]
    a = torch.randn(1100, K, device="cuda").to(torch.bfloat16)
    w_t = (torch.randn(3 * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    d = torch.zeros(1100, N, device="cuda", dtype=torch.bfloat16)
    t = lambda v: torch.tensor(v, dtype=torch.int32, device="cuda")  # noqa: E731
    rs, rw, wi = t(starts), t(rows), t(widx)
    _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), 1100, K, w_t.data_ptr(), 3 * N, N, None,
              d.data_ptr(), 3, rs.data_ptr(), 0, rw.data_ptr(), 0, wi.data_ptr(), 333, 0,
              _lib.stream_ptr())
    torch.cuda.synchronize()
    ref = _ref(a, w_t, None, rows, starts, widx, 0, N)
    for g, want in ref.items():
        got = d[starts[g]:starts[g] + rows[g]].float()
        assert (got - want).abs().max().item() <= 2e-2 * want.abs().max().item()


def test_grouped_gemm_bf16_many_tiles_persistent():
    # more tiles than SMs, uniform groups: exercises the persistent scheduler
    torch.manual_seed(1)
    G, cap, K, N = 16, 640, 1024, 1024
    a = torch.randn(G * cap, K, device="cuda").to(torch.bfloat16)
    w_t = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    d = torch.empty(G * cap, N, device="cuda", dtype=torch.bfloat16)
    _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), G * cap, K, w_t.data_ptr(), G * N, N, None,
              d.data_ptr(), G, None, cap, None, cap, None, cap, 0, _lib.stream_ptr())
    want = torch.bmm(a.view(G, cap, K).float(), w_t.view(G, N, K).float().transpose(1, 2))
    got = d.view(G, cap, N).float()
    assert (got - want).abs().max().item() <= 2e-2 * want.abs().max().item()


@pytest.mark.parametrize("K,N,act", [(1024, 4096, 1), (4096, 1024, 0), (8, 8, 1), (33, 17, 0)])
def test_grouped_gemm_f32(K, N, act):
    torch.manual_seed(K)
    G, cap = 3, 200
    rows = [200, 5, 0]
    a = torch.randn(G * cap, K, device="cuda")
    w = torch.randn(G, K, N, device="cuda") / K ** 0.5
    bias = torch.randn(G, N, device="cuda")
    d = torch.zeros(G * cap, N, device="cuda")
    rows_t = torch.tensor(rows, dtype=torch.int32, device="cuda")
    _lib.call("moe_grouped_gemm_f32", a.data_ptr(), K, w.data_ptr(), N, bias.data_ptr(),
              d.data_ptr(), G, None, cap, rows_t.data_ptr(), 0, None, cap, act, _lib.stream_ptr())
    for g, r in enumerate(rows):
        if r == 0:
            continue
        want = a[g * cap:g * cap + r].double() @ w[g].double() + bias[g].double()
        if act:
            want = _gelu(want)
        got = d[g * cap:g * cap + r].double()
        assert ((got - want).abs() <= 1e-5 * (want.abs() + want.abs().mean())).all()


@pytest.mark.parametrize("P,Q", [(2048, 512), (256, 256), (64, 128), (200, 96), (512, 2048), (136, 264)])
def test_wgrad_bf16(P, Q):
    """Weight-gradient mode (MN-major operands): D[g] = X_g^T Y_g over each
    group's first k_rows[g] rows; rows past k_rows hold NaN and must not leak."""
    torch.manual_seed(P * 7 + Q)
    G, cap = 6, 300
    k_rows = [300, 0, 129, 1, 64, 257]
    x = torch.randn(G * cap, P, device="cuda").to(torch.bfloat16)
    y = torch.randn(G * cap, Q, device="cuda").to(torch.bfloat16)
    for g, r in enumerate(k_rows):
        x[g * cap + r:(g + 1) * cap] = float("nan")
        y[g * cap + r:(g + 1) * cap] = float("nan")
    kr = torch.tensor(k_rows, dtype=torch.int32, device="cuda")
    d = torch.full((G, P, Q), 7.0, dtype=torch.bfloat16, device="cuda")
    _lib.call("moe_grouped_gemm_bf16_wgrad", x.data_ptr(), G * cap, P, y.data_ptr(), Q, G, cap,
              kr.data_ptr(), 0, d.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    for g, r in enumerate(k_rows):
        xs, ys = x[g * cap:g * cap + r].float(), y[g * cap:g * cap + r].float()
        want = xs.t() @ ys
        got = d[g].float()
        assert torch.isfinite(got).all(), g
        tol = 1e-2 * (want.abs() + want.abs().mean() + 1e-3)
        assert ((got - want).abs() <= tol).all(), (g, (got - want).abs().max().item())


@pytest.mark.parametrize("rows,P,Q", [(65536, 2048, 256), (3000, 512, 16), (100, 64, 128), (70000, 1024, 512)])
def test_wgrad_f32_splitk(rows, P, Q):
    torch.manual_seed(rows + P)
    x = torch.randn(rows, P, device="cuda").to(torch.bfloat16)
    y = torch.randn(rows, Q, device="cuda").to(torch.bfloat16)
    d = torch.zeros(P, Q, device="cuda")
    _lib.call("moe_gemm_bf16_wgrad_f32", x.data_ptr(), rows, P, y.data_ptr(), Q, d.data_ptr(),
              _lib.stream_ptr())
    want = x.double().t() @ y.double()
    err = (d.double() - want).abs()
    # fp32 accumulation of exact bf16 products: error ~ rows * eps32 * |x||y|
    assert err.max().item() <= 1e-5 * rows ** 0.5 * 4 + 1e-4 * want.abs().max().item(), err.max().item()


def test_colsum_rows():
    torch.manual_seed(3)
    G, cap, W = 5, 300, 1032
    rows = [300, 0, 129, 1, 257]
    x = torch.randn(G * cap, W, device="cuda").to(torch.bfloat16)
    r = torch.tensor(rows, dtype=torch.int32, device="cuda")
    out = torch.zeros(G, W, device="cuda")
    _lib.call("moe_colsum_rows_bf16", x.data_ptr(), W, G, cap, r.data_ptr(), 0, out.data_ptr(),
              _lib.stream_ptr())
    for g, n in enumerate(rows):
        want = x[g * cap:g * cap + n].double().sum(0)
        assert torch.allclose(out[g].double(), want, atol=1e-3, rtol=1e-5), g


@pytest.mark.parametrize("K,N,act,cap", [(2048, 8192, 1, 512), (1024, 1024, 0, 300), (256, 96, 1, 40),
                                         (136, 200, 0, 129), (512, 4096, 1, 3)])
def test_grouped_gemm_bf16_gather(K, N, act, cap):
    """A rows gathered by index (TMA gather4): equal to the GEMM on the gathered copy."""
    torch.manual_seed(K + N + cap)
    G, S = 5, 700
    rows = [cap, 0, max(cap // 2, 1), 1, min(cap, 257)]
    x = (torch.randn(S, K, device="cuda") * 0.5).to(torch.bfloat16)
    idx = torch.randint(0, S, (G * cap,), dtype=torch.int32, device="cuda")
    w_t = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(G, N, device="cuda") * 0.1
    rows_t = torch.tensor(rows, dtype=torch.int32, device="cuda")
    d = torch.full((G * cap, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    _lib.call("moe_grouped_gemm_bf16_gather", x.data_ptr(), S, idx.data_ptr(), K, w_t.data_ptr(),
              G * N, N, bias.data_ptr(), d.data_ptr(), G, cap, rows_t.data_ptr(), 0, cap,
              act | _lib.MOE_GEMM_PAD_SCRATCH, _lib.stream_ptr())
    # the same GEMM on the materialised gather
    a = x[idx.long()]
    d2 = torch.full_like(d, float("nan"))
    _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), G * cap, K, w_t.data_ptr(), G * N, N,
              bias.data_ptr(), d2.data_ptr(), G, None, cap, rows_t.data_ptr(), 0, None, cap,
              act | _lib.MOE_GEMM_PAD_SCRATCH, _lib.stream_ptr())
    torch.cuda.synchronize()
    for g, r in enumerate(rows):
        got, want = d[g * cap:g * cap + r], d2[g * cap:g * cap + r]
        assert torch.equal(got, want), (g, (got.float() - want.float()).abs().max().item())


@pytest.mark.parametrize("bn512", ["0", "1"])
def test_tile_variants_env(bn512):
    """The expert-GEMM tile choice is read from MOE_BN512 once per process: rerun
    the grouped-GEMM and fused-combine layer parity tests in a child process with
    every 256x512 path forced on (1: bias, bias+GELU at any size, fused combine)
    and with all of them off (0)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MOE_BN512=bn512, PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           "tests/test_gpu_gemm.py::test_grouped_gemm_bf16",
           "tests/test_gpu_layer.py::test_fused_combine_matches_unfused",
           "tests/test_gpu_layer.py::test_bf16_layers_sampled"]
    res = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
