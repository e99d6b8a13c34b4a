"""Stand-alone fused gate at S=65536, M=2048 (E from GATE_E), L2 flushed read-only
before every launch; median of 30. Prints us and HBM GB/s (x bytes)."""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

S, M = 65536, 2048
x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
flush = torch.ones(64 << 20, dtype=torch.int64, device="cuda")  # 512 MB
for E in [int(v) for v in os.environ.get("GATE_E", "128,256,64,16").split(",")]:
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
    ts = []
    for _ in range(30):
        flush.max()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"E={E:4d} {ms * 1e3:7.1f} us  {S * M * 2 / ms / 1e6:7.0f} GB/s")
