"""Time forward_train + backward at a bench workload (default C3); prints the
per-step time. Used for the ncu launch list of the training step."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from bench import WORKLOADS, make_layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
w = WORKLOADS[a.workload]
layer = make_layer(w["S"], w["M"], w["E"], w["k"], w["cf"], torch.device("cuda"),
                   residual=w["residual"])
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(w["S"], w["M"], device="cuda", generator=g).to(torch.bfloat16)
gy = torch.randn(w["S"], w["M"], device="cuda", generator=g).to(torch.bfloat16)
for _ in range(a.warmup):
    layer.forward_train(x)
    layer.backward(gy)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    layer.forward_train(x)
    layer.backward(gy)
e1.record()
torch.cuda.synchronize()
print("train step ms", e0.elapsed_time(e1) / a.steps)
