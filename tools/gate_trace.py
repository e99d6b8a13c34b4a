"""Phase stamps of one gate launch (CTA 0) from the MOE_GATE_TRACE build:
entry, setup done, first TMA issued, first / last K block at the MMA warp,
epilogue start / end of the first tile, teardown, exit. Median of 20 launches,
L2 flushed before each; decode sizes and the C3 batch."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

lib = _lib.load()
fn = lib.moe_debug_gate_trace
fn.argtypes = [ctypes.c_void_p]
M, E = 2048, 128
wg = (torch.randn(E, M, device="cuda") * 0.02).to(torch.bfloat16)
flush = torch.ones(64 << 20, dtype=torch.int64, device="cuda")
names = ["setup", "first TMA", "first full", "last full", "epi start", "epi end", "teardown",
         "exit", "top-k", "sum", "probs", "ranks"]
for S in (16, 64, 512, 65536):
    x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
    ids = torch.empty(S, 1, dtype=torch.int32, device="cuda")
    gp = torch.empty(S, 1, device="cuda")
    lr = torch.empty(S, 1, dtype=torch.int32, device="cuda")
    tc = torch.empty((S + 127) // 128, E, dtype=torch.int32, device="cuda")
    rows = []
    for it in range(23):
        flush.max()
        _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, 1, None, ids.data_ptr(),
                  gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), _lib.stream_ptr())
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 16)()
        fn(buf)
        if it >= 3:
            rows.append([(buf[i] - buf[0]) / 1e3 for i in range(1, 13)])
    med = [sorted(r[i] for r in rows)[len(rows) // 2] for i in range(12)]
    print(f"S={S:6d} " + "  ".join(f"{n} {v:6.1f}" for n, v in zip(names, med)) + "  (us since entry)")
