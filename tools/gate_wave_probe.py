"""Gate wave-quantisation probe: stand-alone fused gate (E=128, k=1, M=2048) at
S = t * 256 tokens for pair-tile counts t around 2, 3, 4 and 5 waves of the 74
SM pairs, L2 flushed read-only before every launch, median of 20; beside it a
plain streaming read of the same x bytes (torch amax over x viewed as int64) as
the achievable read bandwidth. If time(t) steps at multiples of 74 tiles, the
partial last wave costs a full one; if it grows with t, the gate is byte-bound."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

M, E = 2048, 128
flush = torch.ones(64 << 20, dtype=torch.int64, device="cuda")  # 512 MB
wg = (torch.randn(E, M, device="cuda") * 0.02).to(torch.bfloat16)
xs = torch.randn(5 * 74 * 256 + 4096, M, device="cuda").to(torch.bfloat16)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.max()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2] * 1e3


for t in [148, 185, 222, 256, 259, 296, 333, 370]:
    S = t * 256
    x = xs[:S]
    ids = torch.empty(S, 1, dtype=torch.int32, device="cuda")
    gp = torch.empty(S, 1, device="cuda")
    lr = torch.empty(S, 1, dtype=torch.int32, device="cuda")
    tc = torch.empty(S // 128, E, dtype=torch.int32, device="cuda")

    def gate():
        _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, 1, None,
                  ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), _lib.stream_ptr())

    xv = x.view(torch.int64)
    ug = timed(gate)
    ur = timed(lambda: xv.amax())
    b = S * M * 2
    print(f"tiles {t:4d} waves {t / 74:5.2f}  gate {ug:6.1f} us {b / ug / 1e3:6.0f} GB/s"
          f"  | read {ur:6.1f} us {b / ur / 1e3:6.0f} GB/s", flush=True)
