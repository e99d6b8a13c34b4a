"""Host <-> device bandwidth with 1..N GPUs copying at once (one process, one
H2D and one D2H stream per GPU, 268 MB each way per GPU per iteration, pinned
host buffers): the ceiling of bench.py's e2e leg at N > 1."""
import json
import sys
import time

import torch

n = torch.cuda.device_count()
B = 268435456
bufs = []
for d in range(n):
    with torch.cuda.device(d):
        bufs.append(dict(h_in=torch.empty(B, dtype=torch.uint8).pin_memory(),
                         h_out=torch.empty(B, dtype=torch.uint8).pin_memory(),
                         d_in=torch.empty(B, dtype=torch.uint8, device=d),
                         d_out=torch.empty(B, dtype=torch.uint8, device=d),
                         s1=torch.cuda.Stream(device=d), s2=torch.cuda.Stream(device=d)))
res = {}
for g in range(1, n + 1):
    for mode in ("h2d", "d2h", "both"):
        for _ in range(2):  # warm-up + timed
            t0 = time.perf_counter()
            for d in range(g):
                b = bufs[d]
                if mode in ("h2d", "both"):
                    with torch.cuda.stream(b["s1"]):
                        b["d_in"].copy_(b["h_in"], non_blocking=True)
                if mode in ("d2h", "both"):
                    with torch.cuda.stream(b["s2"]):
                        b["h_out"].copy_(b["d_out"], non_blocking=True)
            for d in range(g):
                torch.cuda.synchronize(d)
            dt = time.perf_counter() - t0
        per_dir = B / dt / 1e9  # GB/s per GPU per direction
        res[f"{g}gpu_{mode}"] = round(per_dir, 1)
        print(json.dumps({"gpus": g, "mode": mode, "GB_s_per_gpu_per_direction": round(per_dir, 1),
                          "host_total_GB_s": round(per_dir * g * (2 if mode == "both" else 1), 1)}),
              flush=True)
