"""Per-phase device times of one EP layer forward at decode size (eager, CUDA
events on the launching stream; run under torchrun, one rank per GPU).
python -m torch.distributed.run --nproc-per-node N tools/decode_phases.py [--tokens 64]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402
from paper_2201_05596_b200.ep import EPMoeLayer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=64, help="global tokens")
a = ap.parse_args()
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
W, r = dist.get_world_size(), dist.get_rank()
S = a.tokens // W
layer = EPMoeLayer.synthetic(S, 2048, 128, 1, 1.0, dev, seed=0)
x = torch.randn(S, 2048, device=dev).to(torch.bfloat16)
for _ in range(5):
    layer(x)
torch.cuda.synchronize()
tot = {}
for _ in range(20):
    dist.barrier()
    t = _lib.PhaseTimer()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    layer(x, timer=t)
    e1.record()
    torch.cuda.synchronize()
    for k, v in t.summary(1).items():
        tot.setdefault(k, []).append(v)
    tot.setdefault("total", []).append(e0.elapsed_time(e1))
if r == 0:
    for k, v in tot.items():
        v = sorted(v)
        print(f"{k:20s} median {v[len(v) // 2] * 1e3:8.1f} us")
dist.destroy_process_group()
