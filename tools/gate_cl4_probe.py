"""Gate-GEMM 4-CTA-cluster probe (tuning aid): run once with MOE_GATE_CL4=0 and
once with =1; each run times the fused gate at S=65536, M=2048 (L2 flushed
between launches, E=128 and 256) and saves its routing outputs so the two runs
can be compared bit for bit (``--compare``)."""

import json
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2201_05596_b200 import _lib  # noqa: E402

out_dir = "gpurun_out"
if len(sys.argv) > 1 and sys.argv[1] == "--compare":
    a = torch.load(f"{out_dir}/gate_cl4_0.pt")
    b = torch.load(f"{out_dir}/gate_cl4_1.pt")
    for key in a:
        print(key, "identical" if torch.equal(a[key], b[key]) else "DIFFER")
    sys.exit(0 if all(torch.equal(a[k], b[k]) for k in a) else 1)

mode = os.environ.get("MOE_GATE_CL4", "0")
S, M = 65536, 2048
torch.manual_seed(0)
x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
flush = torch.ones(64 << 20, dtype=torch.int64, device="cuda")  # 512 MB
saved = {}
for E in (128, 256):
    wg = (torch.randn(E, M, device="cuda") * 0.02).to(torch.bfloat16)
    for k in (1, 2):
        ids = torch.empty(S, k, dtype=torch.int32, device="cuda")
        gp = torch.empty(S, k, device="cuda")
        lr = torch.empty(S, k, dtype=torch.int32, device="cuda")
        tc = torch.empty(S // 128, E, dtype=torch.int32, device="cuda")
        logits = torch.empty(S, E, device="cuda")

        def run():
            _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, k,
                      logits.data_ptr(), ids.data_ptr(), gp.data_ptr(), lr.data_ptr(),
                      tc.data_ptr(), _lib.stream_ptr())

        for _ in range(5):
            run()
        torch.cuda.synchronize()
        saved.update({f"E{E}k{k}_{n}": t.clone() for n, t in
                      (("ids", ids), ("gp", gp), ("lr", lr), ("tc", tc), ("logits", logits))})
        _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, k, None,
                  ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), _lib.stream_ptr())
        ts = []
        for _ in range(40):
            flush.max()  # read-only flush: evicts without leaving dirty lines to write back
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("moe_gate_gemm_bf16", x.data_ptr(), wg.data_ptr(), S, M, E, k, None,
                      ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(),
                      _lib.stream_ptr())
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        print(json.dumps({"cl4": int(mode), "E": E, "k": k, "us_p50": round(ms * 1e3, 1),
                          "GB_s": round(S * M * 2 / ms / 1e6)}))
torch.save(saved, f"{out_dir}/gate_cl4_{mode}.pt")
