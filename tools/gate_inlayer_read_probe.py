"""Is the in-layer gate below the HBM roofline because of the gate kernel, or
because of where it runs? C3 layer (65,536 x 2048, 128 experts) on one GPU;
each iteration runs the whole layer forward and then, right behind its GEMM2
(the position the next step's gate occupies), one of:
  gate  - the layer's own fused gate kernel on x (moe_gate_gemm_bf16)
  read  - a plain streaming read of the same 268 MB (torch amax over x as int64)
timed with CUDA events around that kernel alone. The same two kernels are also
timed stand-alone after a read-only 512 MB L2 flush. Prints medians (us) and
GB/s; if `read` behind GEMM2 drops like the gate does, the gate is at the
in-situ read roofline and the gap is the position (clock / power state), not
the kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_05596_b200 import _lib  # noqa: E402

S, M, E = 65536, 2048, 128
dev = torch.device("cuda", 0)
layer = bench.make_layer(S, M, E, 1, 1.0, dev)
x = torch.randn(S, M, device=dev).to(torch.bfloat16)
xv = x.view(torch.int64)
flush = torch.ones(64 << 20, dtype=torch.int64, device=dev)
ws = layer.workspace(S)
ids, gp, lr, tc = (torch.empty_like(ws[n]) for n in ("ids", "gp", "local_rank", "tile_counts"))


def gate():
    _lib.call("moe_gate_gemm_bf16", x.data_ptr(), layer.wg.data_ptr(), S, M, E, 1, None,
              ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), _lib.stream_ptr())


def read():
    xv.amax()


SPIN = 20000  # cycles of torch.cuda._sleep: its event time gives the SM clock at that moment


def timed(fn, behind_layer, reps):
    ts, mhz = [], []
    for _ in range(reps):
        if behind_layer:
            layer(x)
        else:
            flush.amax()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        torch.cuda._sleep(SPIN)
        e1.record()
        fn()
        e2.record()
        torch.cuda.synchronize()
        mhz.append(SPIN / (e0.elapsed_time(e1) * 1e3))
        ts.append(e1.elapsed_time(e2) * 1e3)
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    return med(ts), med(mhz)


for _ in range(3):
    layer(x)
    gate()
    read()
torch.cuda.synchronize()
b = S * M * 2
# alternate the kernels inside every round so both see the same power state
for rnd in range(3):
    for pos in (False, True):
        for name, fn in (("gate", gate), ("read", read)):
            us, mhz = timed(fn, pos, 20)
            where = "behind GEMM2" if pos else "alone, L2 flushed"
            print(f"round {rnd} {name:4s} {where:18s} {us:7.1f} us {b / us / 1e3:6.0f} GB/s "
                  f"{b / us / 1e3 / 6549.4:5.3f} of HBM  SM ~{mhz:5.0f} MHz before it "
                  f"({us * mhz / 1e3:6.0f} kcycles)", flush=True)
