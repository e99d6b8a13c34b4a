"""One workload's layer forward for ncu: W warm-up forwards, then P profiled
forwards (ncu -s skips the warm-up launches: 5 per C3 / C2 step, 4 per grouped
C4 step). python tools/profile_step.py [--workload c3] [--warmup 3] [--steps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--tokens", type=int, default=None, help="tokens (default: the workload's)")
a = ap.parse_args()
wl = dict(bench.WORKLOADS[a.workload])
if a.tokens:
    wl["S"] = a.tokens
dev = torch.device("cuda", 0)
layer = bench.make_layer(wl["S"], wl["M"], wl["E"], wl["k"], wl["cf"], dev, residual=wl["residual"])
x = torch.randn(wl["S"], wl["M"], device=dev, generator=torch.Generator(device=dev).manual_seed(1)
                ).to(torch.bfloat16)
out = torch.empty_like(x)
for _ in range(a.warmup + a.steps):
    layer(x, out=out)
torch.cuda.synchronize()
print("kept", layer.kept_assignments(wl["S"]))
