"""The fused gate (C3: S=65536, M=2048, E=128) timed alone in a loop and right
after a grouped GEMM2 launch (the pipeline position), with SM clocks sampled:
separates the kernel from the power-capped clock state it inherits."""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2201_05596_b200 import _lib  # noqa: E402

S, M, E, G, cap, F = 65536, 2048, 128, 128, 512, 8192
x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
wg = (torch.randn(128, M, device="cuda") * 0.02).to(torch.bfloat16)
ids = torch.empty(S, 1, dtype=torch.int32, device="cuda")
gp = torch.empty(S, 1, device="cuda")
lr = torch.empty(S, 1, dtype=torch.int32, device="cuda")
tc = torch.empty(S // 128, E, dtype=torch.int32, device="cuda")
h = torch.randn(G * cap, F, device="cuda").to(torch.bfloat16)
w2 = (torch.randn(G * M, F, device="cuda") * 0.02).to(torch.bfloat16)
y = torch.empty(G * cap, M, device="cuda", dtype=torch.bfloat16)
b2 = torch.zeros(G, M, device="cuda")
st = _lib.stream_ptr()


def gate():
    _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, 1, None, ids.data_ptr(),
              gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), st)


def gemm2():
    _lib.call("moe_grouped_gemm_bf16", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
              b2.data_ptr(), y.data_ptr(), G, None, cap, None, cap, None, cap, 0, st)


for mode in ("alone", "after_gemm2", "alone"):
    for _ in range(5):
        gate()
    torch.cuda.synchronize()
    ts = []
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                            "-lms", "25"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    t_end = time.time() + 1.5
    while time.time() < t_end:
        if mode == "after_gemm2":
            gemm2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gate()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    smi.terminate()
    clk = sorted(float(v) for v in smi.communicate()[0].split())
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{mode:12s} gate p50 {med * 1e3:6.1f} us  {S * M * 2 / med / 1e6:6.0f} GB/s  "
          f"sm_mhz p50 {clk[len(clk) // 2] if clk else None}")
