"""Burst-clock comparison (GPU idle before each sample): the C3 grouped GEMM1
(bias + GELU, TMA-store epilogue) and plain GEMM2 against cuBLAS torch.bmm with a
distinct weight per expert (the same HBM weight stream), 3 back-to-back launches
after 1 s idle, median of 7 samples of the middle launch. Prints ms and TFLOP/s."""
import json
import os
import sys
import time

import torch

os.environ["PROBE_SET"] = "none"

sys.path.insert(0, ".")
import tools.power_probe as pp  # noqa: E402  (builds the operands; PROBE_SET=none runs nothing)


def sample(fn):
    ts = []
    for _ in range(7):
        torch.cuda.synchronize()
        time.sleep(1.0)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for i in range(3):
            ev[i].record()
            fn()
        ev[3].record()
        torch.cuda.synchronize()
        ts.append(ev[1].elapsed_time(ev[2]))
    return sorted(ts)[3]


fl = 2.0 * pp.G * pp.cap * pp.M * pp.F
for name, fn in (("grouped_gemm1_gelu_tma", pp.g1t), ("cublas_bmm1", pp.bb1),
                 ("grouped_gemm2_fused_combine", pp.g2c), ("grouped_gemm2_tma", pp.g2t),
                 ("cublas_bmm2", pp.bb2)):
    ms = sample(fn)
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}), flush=True)
