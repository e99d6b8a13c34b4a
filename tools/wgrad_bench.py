"""Time the weight-gradient GEMM (MN-major operands) at the C3 expert shape:
E groups of cap rows, D[g] = X_g^T Y_g, with per-group row counts (partial last
K block) vs full groups, against the forward grouped GEMM of equal flops."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05596_b200 import _lib  # noqa: E402

E, cap, M, F = 128, 512, 2048, 8192
g = torch.Generator(device="cuda").manual_seed(0)
h = torch.randn(E * cap, F, device="cuda", generator=g).to(torch.bfloat16)
dy = torch.randn(E * cap, M, device="cuda", generator=g).to(torch.bfloat16)
w2 = torch.randn(E * M, F, device="cuda", generator=g).to(torch.bfloat16)
out = torch.empty(E, F, M, dtype=torch.bfloat16, device="cuda")
yfw = torch.empty(E * cap, M, dtype=torch.bfloat16, device="cuda")
load_partial = torch.randint(cap - 100, cap + 1, (E,), generator=g, device="cuda").to(torch.int32)
st = _lib.stream_ptr()


def run(name, fn, iters=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    print(f"{name:40s} {ms:7.3f} ms  {2.0 * E * cap * M * F / ms / 1e9:7.1f} TF/s")


run("wgrad full groups (K=cap)", lambda: _lib.call(
    "moe_grouped_gemm_bf16_wgrad", h.data_ptr(), E * cap, F, dy.data_ptr(), M, E, cap, None, cap,
    out.data_ptr(), st))
run("wgrad partial groups (k_rows)", lambda: _lib.call(
    "moe_grouped_gemm_bf16_wgrad", h.data_ptr(), E * cap, F, dy.data_ptr(), M, E, cap,
    load_partial.data_ptr(), 0, out.data_ptr(), st))
full = torch.full((E,), cap, dtype=torch.int32, device="cuda")
run("forward GEMM2 (rows=cap, K=F, N=M)", lambda: _lib.call(
    "moe_grouped_gemm_bf16", h.data_ptr(), E * cap, F, w2.data_ptr(), E * M, M, None,
    yfw.data_ptr(), E, None, cap, full.data_ptr(), 0, None, cap, 0, st))
# same tile structure as the wgrad (K = cap), but K-major operands (pre-transposed)
hT = torch.randn(E * F, cap, device="cuda", generator=g).to(torch.bfloat16)
dyT = torch.randn(E * M, cap, device="cuda", generator=g).to(torch.bfloat16)
del w2, yfw
o2 = torch.empty(E * F, M, dtype=torch.bfloat16, device="cuda")
run("K-major short-K GEMM (K=cap)", lambda: _lib.call(
    "moe_grouped_gemm_bf16", hT.data_ptr(), E * F, cap, dyT.data_ptr(), E * M, M, None,
    o2.data_ptr(), E, None, F, None, F, None, F, 0, st))
