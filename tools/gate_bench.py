"""Gate-GEMM microbenchmark (tuning aid): the fused gate kernel alone at
S=65536, M=2048 for several expert counts; reports time and HBM GB/s."""

import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

S, M = 65536, 2048
x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
import os
for E in [int(v) for v in os.environ.get("GATE_E", "8,16,32,64,128,256").split(",")]:
    epad = max(32, 1 << (E - 1).bit_length())
    wg = (torch.randn(epad, M, device="cuda") * 0.02).to(torch.bfloat16)
    ids = torch.empty(S, 1, dtype=torch.int32, device="cuda")
    gp = torch.empty(S, 1, device="cuda")
    lr = torch.empty(S, 1, dtype=torch.int32, device="cuda")
    tc = torch.empty(S // 128, E, dtype=torch.int32, device="cuda")

    def run():
        _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, 1, None,
                  ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), _lib.stream_ptr())

    for _ in range(5):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"E={E:4d} {ms * 1e3:7.1f} us  {S * M * 2 / ms / 1e6:7.0f} GB/s")
