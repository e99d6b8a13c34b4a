"""One launch each of our GEMM1/GEMM2 (C3 expert shape, TMA-store epilogue) and
cuBLAS torch.bmm with per-expert weights, for an ncu DRAM-bytes comparison."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2201_05596_b200 import _lib  # noqa: E402

G, cap, M, F = 128, 512, 2048, 8192
x = torch.randn(G * cap, M, device="cuda").to(torch.bfloat16)
w1 = torch.randn(G * F, M, device="cuda", dtype=torch.bfloat16) * 0.02
w2 = torch.randn(G * M, F, device="cuda", dtype=torch.bfloat16) * 0.02
b1 = torch.zeros(G, F, device="cuda")
b2 = torch.zeros(G, M, device="cuda")
h = torch.empty(G * cap, F, device="cuda", dtype=torch.bfloat16)
y = torch.empty(G * cap, M, device="cuda", dtype=torch.bfloat16)
st = _lib.stream_ptr()
P = _lib.MOE_GEMM_PAD_SCRATCH
for _ in range(2):
    _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), G * cap, M, w1.data_ptr(), G * F, F,
              b1.data_ptr(), h.data_ptr(), G, None, cap, None, cap, None, cap, 1 | P, st)
    _lib.call("moe_grouped_gemm_bf16", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
              b2.data_ptr(), y.data_ptr(), G, None, cap, None, cap, None, cap, 0 | P, st)
    torch.bmm(x.view(G, cap, M), w1.view(G, F, M).transpose(1, 2), out=h.view(G, cap, F))
    torch.bmm(h.view(G, cap, F), w2.view(G, M, F).transpose(1, 2), out=y.view(G, cap, M))
torch.cuda.synchronize()
