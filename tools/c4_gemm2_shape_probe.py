"""C4-32 GEMM2 shape as a plain grouped GEMM (64 groups x 512 rows: 32 experts
+ the shared MLP's 16384 tokens as 32 more groups; K = d_ff 4096, N = d_model
1024), bias epilogue with TMA stores; median of 20 launches after warm-up.
Run twice with MOE_BN512=0 / 3 to see what 256x512 pair tiles buy at this shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

G, cap, K, N = 64, 512, 4096, 1024
a = (torch.randn(G * cap, K, device="cuda") * 0.5).to(torch.bfloat16)
w = (torch.randn(G * N, K, device="cuda") * 0.02).to(torch.bfloat16)
b = torch.zeros(G, N, device="cuda")
d = torch.empty(G * cap, N, device="cuda", dtype=torch.bfloat16)


def run():
    _lib.call("moe_grouped_gemm_bf16", a.data_ptr(), G * cap, K, w.data_ptr(), G * N, N, b.data_ptr(),
              d.data_ptr(), G, None, cap, None, cap, None, cap, _lib.MOE_GEMM_PAD_SCRATCH,
              _lib.stream_ptr())


for _ in range(5):
    run()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[10]
print(f"MOE_BN512={os.environ.get('MOE_BN512', '3')}: {ms * 1e3:.1f} us "
      f"{2 * G * cap * K * N / ms / 1e9:.0f} TFLOP/s")
