"""Clock / power probe: runs a kernel loop for ~2 s while nvidia-smi samples SM
clock and power, for (a) the grouped GEMM1/GEMM2 at C3 and (b) cuBLAS bf16
GEMMs of the same shape (torch.matmul). Prints TFLOP/s with median clock/power."""
import json
import subprocess
import sys
import time

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
# cuBLAS: one big GEMM of the same flops (65536 x 2048 x 8192), weights of one expert
wa = torch.randn(M, F, device="cuda", dtype=torch.bfloat16) * 0.02
wb = torch.randn(F, M, device="cuda", dtype=torch.bfloat16) * 0.02


def g1():
    _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), G * cap, M, w1.data_ptr(), G * F, F,
              b1.data_ptr(), h.data_ptr(), G, None, cap, None, cap, None, cap, 1, st)


def g2():
    _lib.call("moe_grouped_gemm_bf16", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
              b2.data_ptr(), y.data_ptr(), G, None, cap, None, cap, None, cap, 0, st)


def g1t():  # TMA-store epilogue (padding rows are scratch)
    _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), G * cap, M, w1.data_ptr(), G * F, F,
              b1.data_ptr(), h.data_ptr(), G, None, cap, None, cap, None, cap,
              1 | _lib.MOE_GEMM_PAD_SCRATCH, st)


def g2t():
    _lib.call("moe_grouped_gemm_bf16", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
              b2.data_ptr(), y.data_ptr(), G, None, cap, None, cap, None, cap,
              0 | _lib.MOE_GEMM_PAD_SCRATCH, st)


S_tok = G * cap
row_token = torch.randperm(S_tok, device="cuda").to(torch.int32)
row_prob = torch.rand(S_tok, device="cuda")
xres = torch.randn(S_tok, M, device="cuda").to(torch.bfloat16)
outc = torch.empty_like(xres)


def g2c():  # the layer's GEMM2: bias + gate-prob scale + residual combine in the epilogue
    _lib.call("moe_grouped_gemm_bf16_combine", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
              b2.data_ptr(), G, None, cap, None, cap, None, cap, row_token.data_ptr(),
              row_prob.data_ptr(), xres.data_ptr(), outc.data_ptr(), None, st)


def c1():
    torch.matmul(x, wa, out=h)


def c2():
    torch.matmul(h, wb, out=y)


# cuBLAS batched with a distinct weight per expert (the same HBM weight stream as ours)
x3 = x.view(G, cap, M)
h3 = h.view(G, cap, F)
y3 = y.view(G, cap, M)
w1b = w1.view(G, F, M).transpose(1, 2)  # (G, M, F) view of W1^T rows
w2b = w2.view(G, M, F).transpose(1, 2)


def bb1():
    torch.bmm(x3, w1b, out=h3)


def bb2():
    torch.bmm(h3, w2b, out=y3)


def probe(name, fn, secs=2.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    a.record()
    t0 = time.time()
    while time.time() - t0 < secs:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()[4:-2]
    clk = sorted(float(l.split(",")[0]) for l in out)
    pw = sorted(float(l.split(",")[1]) for l in out)
    ms = a.elapsed_time(b) / n
    fl = 2.0 * G * cap * M * F
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1),
                      "sm_mhz_med": clk[len(clk) // 2] if clk else None,
                      "power_w_med": pw[len(pw) // 2] if pw else None,
                      "reasons": sorted({l.split(",")[2].strip() for l in out})}), flush=True)


import os  # noqa: E402

if os.environ.get("PROBE_GEMM_CTAS"):  # cap the persistent GEMM grid (SM-count experiments)
    _lib.call("moe_set_launch_limits", int(os.environ["PROBE_GEMM_CTAS"]), 0)

SETS = {
    "all": (("grouped_gemm1_gelu", g1), ("grouped_gemm1_gelu_tma", g1t), ("cublas_bmm1_per_expert_w", bb1),
            ("grouped_gemm2", g2), ("grouped_gemm2_tma", g2t), ("cublas_bmm2_per_expert_w", bb2),
            ("grouped_gemm1_gelu", g1), ("grouped_gemm1_gelu_tma", g1t)),
    "ab": (("grouped_gemm1_gelu_tma", g1t), ("grouped_gemm2_tma", g2t)),
    "cmp": (("grouped_gemm1_gelu_tma", g1t), ("cublas_bmm1_per_expert_w", bb1),
            ("grouped_gemm2_fused_combine", g2c), ("grouped_gemm2_tma", g2t),
            ("cublas_bmm2_per_expert_w", bb2)) * 2,
}
SETS["g2c"] = (("grouped_gemm2_fused_combine", g2c), ("grouped_gemm2_tma", g2t)) * 2
SETS["none"] = ()  # (operands only: tools/burst_vs_cublas.py imports this module)
for name, fn in SETS[os.environ.get("PROBE_SET", "all")]:
    probe(name, fn)
    time.sleep(1.0)
