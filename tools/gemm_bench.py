"""Grouped expert-GEMM microbenchmark at the C3 shape (tuning aid, not the
headline bench). Runs each MOE_GEMM_VARIANT in its own process, interleaved,
and prints TFLOP/s for GEMM1 (bias+GELU) and GEMM2 (bias).

    python tools/gemm_bench.py [--variants 0,1,2] [--rounds 2]
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(iters: int) -> None:
    sys.path.insert(0, ROOT)
    import torch

    from paper_2201_05596_b200 import _lib

    G, cap, M, F = 128, 512, 2048, 8192
    dev = "cuda"
    x = torch.randn(G * cap, M, device=dev).to(torch.bfloat16)
    w1 = (torch.randn(G * F, M, device=dev, dtype=torch.bfloat16) * 0.02)
    w2 = (torch.randn(G * M, F, device=dev, dtype=torch.bfloat16) * 0.02)
    b1 = torch.zeros(G, F, device=dev)
    b2 = torch.zeros(G, M, device=dev)
    h = torch.empty(G * cap, F, device=dev, dtype=torch.bfloat16)
    y = torch.empty(G * cap, M, device=dev, dtype=torch.bfloat16)
    st = _lib.stream_ptr()

    def g1():
        _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), G * cap, M, w1.data_ptr(), G * F, F,
                  b1.data_ptr(), h.data_ptr(), G, None, cap, None, cap, None, cap, 1, st)

    def g2():
        _lib.call("moe_grouped_gemm_bf16", h.data_ptr(), G * cap, F, w2.data_ptr(), G * M, M,
                  b2.data_ptr(), y.data_ptr(), G, None, cap, None, cap, None, cap, 0, st)

    for _ in range(3):
        g1(); g2()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t1 = t2 = 0.0
    for _ in range(iters):
        ev[0].record(); g1(); ev[1].record(); g2(); ev[2].record()
        torch.cuda.synchronize()
        t1 += ev[0].elapsed_time(ev[1]); t2 += ev[1].elapsed_time(ev[2])
    fl = 2.0 * G * cap * M * F
    print(json.dumps({"variant": {k: v for k, v in os.environ.items() if k.startswith("MOE_")},
                      "gemm1_ms": t1 / iters, "gemm2_ms": t2 / iters,
                      "gemm1_tflops": fl / (t1 / iters) / 1e9, "gemm2_tflops": fl / (t2 / iters) / 1e9}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="0,1,2")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--env", default="MOE_GEMM_VARIANT", help="env var the variants set")
    a = ap.parse_args()
    if a.child:
        child(a.iters)
        return
    for _ in range(a.rounds):
        for v in a.variants.split(","):
            env = dict(os.environ, **{a.env: v})
            out = subprocess.run([sys.executable, __file__, "--child", "--iters", str(a.iters)],
                                 env=env, capture_output=True, text=True)
            print(out.stdout.strip() or out.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()
