"""NVLink evidence for the expert-parallel peer-memory kernels, in ONE process
driving two GPUs (ncu must not wrap a multi-rank command; this is one rank
playing both sides). The two "ranks" run exactly the EP layer's p2p data path
(ep.EPMoeLayer._forward_p2p) with the host standing in for the flag barriers:

  gate + local counts (each GPU) -> (host) counts of both ranks -> moe_ep_plan
  -> plan scan with the rank prefixes -> moe_dispatch_p2p (rows stored into
  the owner's receive buffer on the other GPU over NVLink) -> GEMM1 on each
  owner -> moe_grouped_gemm_bf16_push (combined rows stored straight into the
  source's output over NVLink).

Checks the outputs against the single-GPU layer on the concatenated batch
(bit-identical), then prints per-phase device times. Under
  ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,... -k regex:"scatter|gemm_bf16"
the dispatch and push-GEMM launches carry the NVLink tx/rx byte counters.

python tools/nvlink_ep_probe.py [--tokens 65536] [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_05596_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=65536, help="tokens per rank")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
assert torch.cuda.device_count() >= 2, "needs two GPUs"
S, M, E, k, cf = a.tokens, 2048, 128, 1, 1.0
F, W = 4 * M, 2
EL = E // W
devs = [torch.device("cuda", r) for r in range(W)]
lib = _lib.load()
for r in range(W):
    torch.cuda.set_device(r)
    _lib.check(lib.moe_enable_peer_access(1 - r), "moe_enable_peer_access")
torch.cuda.set_device(0)

# single-GPU reference layer on GPU 0 (also the source of the sharded weights)
full = bench.make_layer(S * W, M, E, k, cf, devs[0])
gen = torch.Generator(device=devs[0]).manual_seed(5)
x_all = torch.randn(S * W, M, device=devs[0], generator=gen).to(torch.bfloat16)
want = full(x_all).clone()
cap = full.spec.gating.capacity(S * W)
rmax = EL * cap
i32 = dict(dtype=torch.int32)
T = (S + 127) // 128

R = []
for r, d in enumerate(devs):
    with torch.cuda.device(d):
        st = dict(
            x=x_all[r * S:(r + 1) * S].to(d), wg=full.wg.to(d),
            w1=full.w1[r * EL * F:(r + 1) * EL * F].to(d), w2=full.w2[r * EL * M:(r + 1) * EL * M].to(d),
            b1=full.b1[r * EL:(r + 1) * EL].to(d), b2=full.b2[r * EL:(r + 1) * EL].to(d),
            ids=torch.empty((S, k), device=d, **i32), gp=torch.empty((S, k), device=d),
            lr=torch.empty((S, k), device=d, **i32), tc=torch.empty((T, E), device=d, **i32),
            tof=torch.empty((T, E), device=d, **i32), tot=torch.empty(E, device=d, **i32),
            kept=torch.empty(E, device=d, **i32), slots=torch.empty((S, k), device=d, **i32),
            rix=torch.empty((S, k), device=d, **i32),
            slot_base=torch.empty(E, device=d, **i32), row_base=torch.empty(E, device=d, **i32),
            seg_start=torch.empty(EL, device=d, **i32), seg_rows=torch.empty(EL, device=d, **i32),
            seg_w=torch.arange(EL, device=d, dtype=torch.int32), recv_rows=torch.empty(1, device=d, **i32),
            recv=torch.empty((rmax, M), device=d, dtype=torch.bfloat16),
            row_token=torch.empty(rmax, device=d, **i32), row_prob=torch.empty(rmax, device=d),
            row_src=torch.empty(rmax, device=d, **i32),
            h=torch.empty((rmax, F), device=d, dtype=torch.bfloat16),
            out=torch.empty((S, M), device=d, dtype=torch.bfloat16),
        )
        R.append(st)
for r, d in enumerate(devs):  # peer pointer tables, resident on each GPU
    with torch.cuda.device(d):
        for name in ("recv", "row_token", "row_prob", "row_src", "out"):
            R[r]["peer_" + name] = torch.tensor([R[q][name].data_ptr() for q in range(W)],
                                                dtype=torch.int64, device=d)


def sync():
    for d in devs:
        torch.cuda.synchronize(d)


def step(timers=None):
    ev = {}

    def mark(r, name):
        if timers is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev.setdefault(r, []).append((name, e))

    for r, d in enumerate(devs):
        with torch.cuda.device(d):
            s = R[r]
            st_ = _lib.stream_ptr()
            mark(r, "gate")
            _lib.call("moe_gate_gemm_bf16", s["x"].data_ptr(), s["wg"].data_ptr(), S, M, E, k, None,
                      s["ids"].data_ptr(), s["gp"].data_ptr(), s["lr"].data_ptr(), s["tc"].data_ptr(), st_)
            _lib.call("moe_plan_scan", s["tc"].data_ptr(), S, E, 2 ** 62, None, s["tof"].data_ptr(),
                      s["tot"].data_ptr(), s["kept"].data_ptr(), st_)
    sync()  # (the layer all-gathers the counts over peer memory here)
    counts = torch.cat([R[q]["tot"].cpu() for q in range(W)])
    for r, d in enumerate(devs):
        with torch.cuda.device(d):
            s = R[r]
            st_ = _lib.stream_ptr()
            cnt = counts.to(d)
            s["_cnt"] = cnt
            mark(r, "plan")
            _lib.call("moe_ep_plan_padded", cnt.data_ptr(), W, r, E, cap, s["slot_base"].data_ptr(),
                      s["row_base"].data_ptr(), s["seg_start"].data_ptr(), s["seg_rows"].data_ptr(),
                      s["recv_rows"].data_ptr(), st_)
            _lib.call("moe_plan_scan", s["tc"].data_ptr(), S, E, cap, s["slot_base"].data_ptr(),
                      s["tof"].data_ptr(), s["tot"].data_ptr(), s["kept"].data_ptr(), st_)
            mark(r, "dispatch_p2p")
            _lib.call("moe_dispatch_p2p", s["x"].data_ptr(), S, M * 2, E, k, cap, s["ids"].data_ptr(),
                      s["lr"].data_ptr(), s["tof"].data_ptr(), s["gp"].data_ptr(),
                      s["slot_base"].data_ptr(), s["row_base"].data_ptr(), EL,
                      s["peer_recv"].data_ptr(), s["peer_row_token"].data_ptr(),
                      s["peer_row_prob"].data_ptr(), s["slots"].data_ptr(), s["rix"].data_ptr(),
                      s["out"].data_ptr(), s["peer_row_src"].data_ptr(), r, st_)
            mark(r, "end_dispatch")
    sync()  # (flag barrier)
    for r, d in enumerate(devs):
        with torch.cuda.device(d):
            s = R[r]
            st_ = _lib.stream_ptr()
            mark(r, "gemm1")
            _lib.call("moe_grouped_gemm_bf16", s["recv"].data_ptr(), rmax, M, s["w1"].data_ptr(), EL * F,
                      F, s["b1"].data_ptr(), s["h"].data_ptr(), EL, None, cap,
                      s["seg_rows"].data_ptr(), 0, None, cap,
                      _lib.MOE_ACT_GELU | _lib.MOE_GEMM_PAD_SCRATCH, st_)
            mark(r, "gemm2_push")
            _lib.call("moe_grouped_gemm_bf16_push", s["h"].data_ptr(), rmax, F, s["w2"].data_ptr(),
                      EL * M, M, s["b2"].data_ptr(), EL, None, cap,
                      s["seg_rows"].data_ptr(), None, cap, 1,
                      s["row_token"].data_ptr(), s["row_prob"].data_ptr(), s["row_src"].data_ptr(),
                      s["peer_out"].data_ptr(), s["recv"].data_ptr(), st_)
            mark(r, "end")
    sync()  # (flag barrier)
    if timers is not None:
        for r in range(W):
            lst = ev[r]
            for (n0, e0), (n1, e1) in zip(lst[:-1], lst[1:]):
                if n0 in ("end_dispatch",):
                    continue
                timers.setdefault(f"rank{r}_{n0}", []).append(e0.elapsed_time(e1))


step()
for r in range(W):
    got = R[r]["out"].to(devs[0])
    ok = torch.equal(got, want[r * S:(r + 1) * S])
    print(f"rank {r}: output bit-identical to the single-GPU layer: {ok}")
    assert ok
timers = {}
for _ in range(a.iters):
    step(timers)
kept = [int(R[r]["seg_rows"].sum().item()) for r in range(W)]
print("received rows per owner:", kept)
for key, v in sorted(timers.items()):
    v = sorted(v)
    print(f"{key:28s} median {v[len(v) // 2]:.4f} ms")
# rows crossing NVLink each way (owner != source): dispatch rows and returned rows
for r in range(W):
    ids = R[r]["ids"][:, 0]
    sl = R[r]["slots"][:, 0]
    remote = int(((ids // EL != r) & (sl >= 0)).sum().item())
    print(f"rank {r}: {remote} kept rows to the other GPU = {remote * M * 2 / 1e6:.1f} MB each way")
