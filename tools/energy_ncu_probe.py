"""Per-launch activity counters of our grouped GEMM2 / GEMM1 against cuBLAS's
batched GEMM of the same C3 expert shape, for an ncu metrics pass (instructions
issued, L2 / shared-memory traffic, DRAM bytes): both kernels settle at the
1 kW power cap, ours at a ~10% lower clock (profiles/r1_power_probe.json), so
the activity per flop is what differs. Run under
  ncu --metrics <list> --kernel-name regex:"gemm_bf16_tc|nvjet" python tools/energy_ncu_probe.py
"""
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
pad = _lib.MOE_GEMM_PAD_SCRATCH
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), G * cap, M, w1.data_ptr(), G * F, F,
              b1.data_ptr(), h.data_ptr(), G, None, cap, None, cap, None, cap, 1 | pad, st)
    _lib.call("moe_grouped_gemm_bf16", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
              b2.data_ptr(), y.data_ptr(), G, None, cap, None, cap, None, cap, 0 | pad, st)
    torch.bmm(x.view(G, cap, M), w1.view(G, F, M).transpose(1, 2), out=h.view(G, cap, F))
    torch.bmm(h.view(G, cap, F), w2.view(G, M, F).transpose(1, 2), out=y.view(G, cap, M))
torch.cuda.synchronize()
print("ok")
