"""Host<->device copy bandwidth with pinned memory: one stream vs the same bytes
split over 2 / 4 streams, each direction alone and both at once (the e2e path
moves 268 MB each way per C3 step)."""
import json

import torch

NB = 256 << 20
h_in = torch.empty(NB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(NB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(NB, dtype=torch.uint8, device="cuda")
d_out = torch.empty(NB, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(nstreams, h2d, d2h, iters=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for _ in range(iters):
        ev = torch.cuda.Event()
        ev.record(cur)
        n = NB // nstreams
        for i in range(nstreams):
            if h2d:
                s = streams[i]
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    d_in[i * n:(i + 1) * n].copy_(h_in[i * n:(i + 1) * n], non_blocking=True)
            if d2h:
                s = streams[4 + i % 4] if h2d else streams[i]
                s.wait_event(ev)
                with torch.cuda.stream(s):
                    h_out[i * n:(i + 1) * n].copy_(d_out[i * n:(i + 1) * n], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return round(NB / ms / 1e6, 1)


res = {}
for ns in (1, 2, 4):
    res[f"h2d_{ns}"] = run(ns, True, False)
    res[f"d2h_{ns}"] = run(ns, False, True)
    res[f"both_{ns}"] = run(ns, True, True)
print(json.dumps({"GB_s_per_direction": res}))
