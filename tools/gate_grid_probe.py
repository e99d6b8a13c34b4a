"""Gate-GEMM grid probe (tuning aid): the fused gate kernel at S=65536, M=2048,
E=128 (C3) with the persistent grid capped at several CTA counts
(moe_set_launch_limits), to see whether the 3.46-wave tail of 256 pair tiles
over 74 clusters costs HBM bandwidth. Prints one JSON line per cap."""

import json
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

S, M, E = 65536, 2048, 128
x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
wg = (torch.randn(E, M, device="cuda") * 0.02).to(torch.bfloat16)
ids = torch.empty(S, 1, dtype=torch.int32, device="cuda")
gp = torch.empty(S, 1, device="cuda")
lr = torch.empty(S, 1, dtype=torch.int32, device="cuda")
tc = torch.empty(S // 128, E, dtype=torch.int32, device="cuda")
flush = torch.ones(64 << 20, dtype=torch.int64, device="cuda")  # 512 MB


def run():
    _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, 1, None,
              ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), _lib.stream_ptr())


ref = None
for cap in [0, 148, 144, 136, 128, 120, 112, 96, 0]:
    _lib.call("moe_set_launch_limits", cap, 0)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    if ref is None:
        ref = ids.clone()
    assert torch.equal(ids, ref)
    ts = []
    for _ in range(30):
        flush.max()  # read-only flush: evicts without leaving dirty lines to write back
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(json.dumps({"cta_cap": cap, "us_p50": round(ms * 1e3, 1),
                      "GB_s": round(S * M * 2 / ms / 1e6)}))
_lib.call("moe_set_launch_limits", 0, 0)
