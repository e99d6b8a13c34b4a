"""Combine-kernel microbenchmark (tuning aid) at the C2 (k=2) and C4 (residual) shapes."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

for name, S, M, E, k, cap, res in [("c2", 16384, 1024, 16, 2, 2560, False),
                                    ("c4", 16384, 1024, 32, 1, 512, True),
                                    ("c3-unfused", 65536, 2048, 128, 1, 512, False)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    ids = torch.stack([torch.randperm(E, device="cuda", generator=g)[:k] for _ in range(1)]).repeat(S, 1)
    ids = torch.randint(0, E, (S, k), device="cuda", generator=g, dtype=torch.int32)
    if k == 2:
        ids[:, 1] = (ids[:, 0] + 1) % E
    slots = torch.randint(0, cap, (S, k), device="cuda", generator=g, dtype=torch.int32)
    gp = torch.rand(S, k, device="cuda")
    y = torch.randn(E * cap, M, device="cuda").to(torch.bfloat16)
    x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
    sh = torch.randn(S, M, device="cuda").to(torch.bfloat16) if res else None
    out = torch.empty_like(x)

    def run():
        _lib.call("moe_combine", y.data_ptr(), _lib.MOE_BF16, S, M, E, k, cap, ids.data_ptr(),
                  slots.data_ptr(), None, gp.data_ptr(), _lib.MOE_F32, x.data_ptr(),
                  _lib.ptr(sh), out.data_ptr(), 1, _lib.stream_ptr())

    for _ in range(5):
        run()
    torch.cuda.synchronize()
    flush = torch.ones(64 << 20, dtype=torch.int64, device="cuda")  # 512 MB
    ts = []
    for _ in range(30):  # L2 flushed before every launch, median
        flush.max()  # read-only flush: evicts without leaving dirty lines to write back
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    nbytes = S * M * 2 * (k + 2 + (1 if res else 0))
    print(f"{name}: {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s")
