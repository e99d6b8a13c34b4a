"""MoE-layer forward benchmark (BASELINE.json metric: tokens/s at the
1.3B+MoE-128 layer shape on 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step is one full MoE-layer forward (gate GEMM + routing epilogue, capacity
scan, dispatch, grouped expert GEMM1/GEMM2, combine + residual) over one batch
of synthetic tokens already resident in HBM. N=1 runs BASELINE config 3 on one
GPU (S=65536, d_model=2048, d_ff=8192, 128 experts, top-1, cf=1.0, bf16).
N>1 (torchrun, one rank per GPU, NCCL) runs the expert-parallel layer with
S=65536 tokens per rank (weak scaling: global batch 65536*N, global capacity).

``--impl reference`` times the reference algorithm on the host CPU: the CPU
oracle (oracle/moe_oracle.py, a float64 NumPy restatement of moekit's
forward_layer) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer fwd tokens/s @1.3B+MoE-128 shape"
UNIT = "tokens/s"
C3 = dict(S=65536, M=2048, E=128, k=1, cf=1.0)
# BASELINE.json configs as bench workloads (c3 is the headline / default)
WORKLOADS = {
    "c3": dict(S=65536, M=2048, E=128, k=1, cf=1.0, residual=False,
               desc="C3: 1.3B+MoE-128 MoE layer (d_model 2048, d_ff 8192, 128 experts, top-1, cf 1.0)"),
    "c2": dict(S=16384, M=1024, E=16, k=2, cf=1.25, residual=False,
               desc="C2: top-2, cf 1.25 with drops, 16 experts, d_model 1024, 16384 tokens"),
    "c4-32": dict(S=16384, M=1024, E=32, k=1, cf=1.0, residual=True,
                  desc="C4: 350M+PR-MoE-32/64 layer with 32 experts + Residual-MoE shared MLP"),
    "c4-64": dict(S=16384, M=1024, E=64, k=1, cf=1.0, residual=True,
                  desc="C4: 350M+PR-MoE-32/64 layer with 64 experts + Residual-MoE shared MLP"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (default: workload's)")
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--decode-iters", type=int, default=50)
    ap.add_argument("--train-steps", type=int, default=10)
    ap.add_argument("--no-decode-graph", dest="decode_graph", action="store_false")
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                    help="N>1 exchange transport (auto: peer memory for k=1 layers)")
    ap.add_argument("--schedule", default="flat", choices=["flat", "hierarchical"],
                    help="N>1 nccl all-to-all schedule (commsim.py:239-370)")
    ap.add_argument("--chunks", type=int, default=1,
                    help="N>1 p2p: token chunks pipelined through dispatch / GEMMs / pull")
    ap.add_argument("--comm-sms", type=int, default=16,
                    help="SMs the GEMMs leave to the copy kernels when chunked")
    ap.add_argument("--gpus-per-node", type=int, default=None,
                    help="node size for --schedule hierarchical (default N/2)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of moekit.arch.forward_layer)
# ---------------------------------------------------------------------------

CPU_SAMPLE = dict(S=2048, M=2048, E=4, k=1, cf=1.0)  # 4 experts x cap 512 of the C3 expert shape


def cpu_reference_step(state=None):
    from oracle import moe_oracle as O

    if state is None:
        s = CPU_SAMPLE
        rng = np.random.default_rng(0)
        gw, experts, _ = O.init_layer_params(s["M"], s["E"], False, rng)
        x = rng.standard_normal((s["S"], s["M"]))
        state = (x, gw, experts)
    x, gw, experts = state
    t0 = time.perf_counter()
    O.forward_layer(x, gw, experts, None, CPU_SAMPLE["E"], CPU_SAMPLE["k"], CPU_SAMPLE["cf"])
    return time.perf_counter() - t0, state


def cpu_desc():
    s = CPU_SAMPLE
    return (f"oracle forward_layer (float64 NumPy/OpenBLAS) on {s['S']} tokens x {s['E']} experts "
            f"of the C3 expert shape (d_model {s['M']}, d_ff {4 * s['M']}, top-1, cf 1.0 -> "
            f"capacity 512 = the C3 per-expert load)")


def _all_blas_threads() -> int:
    """Use every host core for the CPU legs: torchrun exports OMP_NUM_THREADS=1,
    which OpenBLAS read at import; threadpoolctl lifts it at run time."""
    cores = len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=cores)
    except Exception:  # noqa: BLE001 - keep whatever the BLAS was started with
        pass
    return cores


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = _all_blas_threads()
    times, state = [], None
    # each step is ~1.3 s of CPU work: the timed steps stop once ~150 s are spent so
    # the arm ends within a few minutes whatever --steps is (the line reports both)
    t_start = None
    for i in range(args.warmup + args.steps):
        dt, state = cpu_reference_step(state)
        if i >= args.warmup:
            times.append(dt)
            t_start = t_start or time.time() - dt
            if time.time() - t_start > 150.0:
                break
    med = statistics.median(times)
    value = CPU_SAMPLE["S"] / med
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "steps_requested": args.steps,
        "warmup": args.warmup,
        "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS["c3"]["desc"], "tokens_per_gpu": WORKLOADS["c3"]["S"],
                   "global_batch": WORKLOADS["c3"]["S"] * args.gpus, "parallelism": "cpu",
                   "sample": {"tokens": CPU_SAMPLE["S"], "experts": CPU_SAMPLE["E"],
                              "note": "bounded sample of the same layer shape (per-expert load "
                                      "= the C3 capacity 512); tokens/s is per token either way"}},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": cpu_desc()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampler (every 25 ms), started before the warm-up so it is up
    when the timed region begins; only samples stamped inside [mark(), stop()]
    are kept."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        self.idx = gpu_index
        self.t0 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "25"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def mark(self) -> None:
        self.t0 = time.time()

    def stop(self) -> dict:
        import datetime

        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        stamped = []
        for line in open(self.f.name):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                stamped.append((ts, (float(parts[1]), float(parts[2]), parts[5:9])))
            except ValueError:
                continue
        os.unlink(self.f.name)
        t0 = self.t0 if self.t0 is not None else -float("inf")
        rows = [r for ts, r in stamped if t0 <= ts <= t1]
        note = None
        if not rows:
            # a timed region shorter than nvidia-smi's effective sampling period:
            # report the samples taken within 250 ms of it
            rows = [r for ts, r in stamped if t0 - 0.25 <= ts <= t1 + 0.25]
            note = "no sample inside the timed region; samples within 250 ms of it"
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        mx = max(r[1] for r in rows)
        loaded = [r for r in rows if r[0] > 0.5 * mx] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v == "Active"})
        out = {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": mx,
               "reasons": reasons, "samples": len(rows)}
        if note:
            out["note"] = note
        return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def make_layer(S, M, E, k, cf, dev, seed=0, residual=False):
    import torch

    from paper_2201_05596_b200 import arch as A
    from paper_2201_05596_b200.gating import GatingConfig

    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=residual,
                       gating=GatingConfig(E, k, cf))
    gen = torch.Generator(device=dev).manual_seed(seed)
    F = 4 * M
    # random-init weights of the named architecture: N(0,1)*0.1, zero biases (arch.py:347-365)
    gw = torch.randn(M, E, device=dev, generator=gen) * 0.1
    w1 = torch.randn(E, M, F, device=dev, generator=gen, dtype=torch.bfloat16) * 0.1
    w2 = torch.randn(E, F, M, device=dev, generator=gen, dtype=torch.bfloat16) * 0.1
    zb1, zb2 = torch.zeros(1, F, device=dev), torch.zeros(1, M, device=dev)
    shared = None
    if residual:
        shared = A.FfnParams(torch.randn(M, F, device=dev, generator=gen, dtype=torch.bfloat16) * 0.1,
                             zb1, torch.randn(F, M, device=dev, generator=gen,
                                              dtype=torch.bfloat16) * 0.1, zb2)
    p = A.MoeLayerParams(gate_w=gw, experts=tuple(A.FfnParams(w1[e], zb1, w2[e], zb2)
                                                   for e in range(E)), shared=shared)
    layer = A.MoeLayer(spec, p, dtype=torch.bfloat16, device=dev)
    del w1, w2, p
    torch.cuda.empty_cache()
    return layer


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2201_05596_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = WORKLOADS[args.workload]
    S = args.tokens or wl["S"]
    M, E, k, cf, residual = wl["M"], wl["E"], wl["k"], wl["cf"], wl["residual"]
    F = 4 * M
    if world > 1:
        from paper_2201_05596_b200.ep import EPMoeLayer

        gpn = args.gpus_per_node or max(world // 2, 1)
        layer = EPMoeLayer.synthetic(S, M, E, k, cf, dev, seed=0, residual=residual,
                                     transport=args.transport, schedule=args.schedule,
                                     gpus_per_node=gpn if args.schedule == "hierarchical" else None,
                                     chunks=args.chunks, comm_sms=args.comm_sms)
    else:
        layer = make_layer(S, M, E, k, cf, dev, residual=residual)
    gen = torch.Generator(device=dev).manual_seed(1 + rank)
    x = torch.randn(S, M, device=dev, generator=gen).to(torch.bfloat16)
    # drop-free synthetic routing at C3 with unbiased logits is ~1.9% drops
    out = torch.empty_like(x)
    clocks = Clocks(local) if rank == 0 else None
    for _ in range(args.warmup):
        layer(x, out=out)
    torch.cuda.synchronize()

    # ---- timed region: K full forwards, inputs resident (x 268 MB + weights 8.6 GB >> L2)
    timer = _lib.PhaseTimer()
    launches0 = _lib.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.mark()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        layer(x, out=out, timer=timer)
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps
    launches = _lib.launch_count() - launches0
    clk = clocks.stop() if clocks else None
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    phases = timer.summary(args.steps)
    kept = int(layer.kept_assignments(S)) if hasattr(layer, "kept_assignments") else S * k
    # ---- decode (BASELINE config 5): p50 latency of one layer forward for small
    # global batches at the same layer shape (weights streamed from HBM)
    decode = {}
    decode_roof = {}
    if not args.no_decode:
        for sd in (64, 128, 256, 512):
            s_loc = sd // world
            xd = torch.randn(s_loc, M, device=dev, generator=gen).to(torch.bfloat16)
            # decode runs the layer as one CUDA graph (launch-bound sizes)
            graph_ok = world == 1 or getattr(layer, "transport", "") == "p2p"
            fwd = layer.graphed(s_loc) if (args.decode_graph and graph_ok) else layer
            for _ in range(3):
                fwd(xd)
            lat = []
            for _ in range(args.decode_iters):
                if world > 1:
                    dist.barrier()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record()
                fwd(xd)
                a1.record()
                a1.synchronize()
                lat.append(a0.elapsed_time(a1))
            lt = torch.tensor(lat, device=dev)
            if world > 1:
                dist.all_reduce(lt, op=dist.ReduceOp.MAX)
            decode[str(sd)] = round(float(lt.median().item()), 4)
            if world == 1:  # weight bytes the batch actually streams (experts with load > 0)
                load = layer.plan(s_loc)[3]
                active = int((load > 0).sum().item())
                wbytes = active * (2 * M * F * 2 + (F + M) * 4)
                decode_roof[str(sd)] = {"active_experts": active, "weight_bytes": wbytes,
                                        "GB_s": round(wbytes / (decode[str(sd)] * 1e-3) / 1e9, 1)}
    # ---- training step (forward saving context + backward), N=1 only: reported
    # beside the inference metric; 12*A*M*F GEMM flops per step
    train = None
    if world == 1 and args.train_steps > 0 and hasattr(layer, "forward_train"):
        gy = torch.randn(S, M, device=dev, generator=gen).to(torch.bfloat16)
        for _ in range(3):
            layer.forward_train(x)
            layer.backward(gy)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.train_steps + 1)]
        gc.disable()  # no collector pauses between the host-side launches of a step
        ev[0].record()
        for i in range(args.train_steps):
            layer.forward_train(x)
            layer.backward(gy)
            ev[i + 1].record()
        torch.cuda.synchronize()
        gc.enable()
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.train_steps)]
        tms = ev[0].elapsed_time(ev[-1]) / args.train_steps
        train = {"ms_per_step": round(tms, 3), "ms_per_step_median": round(statistics.median(per), 3),
                 "tokens_per_s": S / (tms * 1e-3),
                 "gemm_tflops": 12.0 * kept * M * F / (tms * 1e-3) / 1e12,
                 "steps": args.train_steps, "note": "forward_train + backward, bf16"}
        layer._train_ctx = None
        torch.cuda.empty_cache()
    # ---- e2e through the public API: pinned host x -> layer(x) -> pinned host out.
    # Each step uploads its 268 MB batch and downloads its 268 MB result; the
    # layer streams host batches (H2D / forward / D2H overlapped across steps).
    xh = x.cpu().pin_memory()
    ohs = [torch.empty_like(xh).pin_memory() for _ in range(2)]
    for i in range(2):
        layer(xh, out=ohs[i % 2])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        layer(xh, out=ohs[i % 2])
    layer._pipe.wait()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        kt = torch.tensor([kept], device=dev, dtype=torch.int64)
        dist.all_reduce(kt)
        kept_total = int(kt.item())
    else:
        kept_total = kept

    if rank != 0:
        dist.destroy_process_group()
        return
    hbm, tf_burst, tf_sus, src = peaks()
    # dominant kernel: the grouped expert GEMM (GEMM1 + GEMM2 launches)
    gemm_ms = sum(v for kk, v in phases.items() if kk.startswith("gemm") or kk == "shared_mlp")
    kept_rank = kept_total / world
    # 2*A*M*F per expert GEMM launch (two launches), + 4*S*M*F for the shared MLP
    flops = 4.0 * kept_rank * M * F + (4.0 * S * M * F if residual else 0.0)
    achieved = flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("grouped_gemm_bytes_per_step")
    cpu = None
    if world == 1 and not args.no_cpu_baseline and args.workload == "c3":
        cores = _all_blas_threads()
        _, state = cpu_reference_step()  # warm-up (BLAS threads, page faults)
        dts = [cpu_reference_step(state)[0] for _ in range(3)]
        cpu = {"value": CPU_SAMPLE["S"] / statistics.median(dts), "unit": UNIT, "cores": cores,
               "kind": "port", "sample": cpu_desc() + "; median of 3 after one warm-up"}
    # HBM-bound components (SURVEY 8(d) formulas, per rank, phase times from the
    # timed region): achieved GB/s and fraction of the measured HBM peak
    A_r = kept_rank
    T_r = (S + 127) // 128
    epad = max(32, 1 << (E - 1).bit_length())
    comp_bytes = {"gate": S * M * 2 + epad * M * 2 + S * k * 12 + T_r * E * 4,
                  "dispatch": 2 * A_r * M * 2,
                  "combine": (A_r * M + 2 * S * M + (S * M if residual else 0)) * 2}
    components = {}
    for name, nbytes in comp_bytes.items():
        t_ms = phases.get(name)
        if t_ms:
            gbs = nbytes / (t_ms * 1e-3) / 1e9
            components[name] = {"ms": round(t_ms, 4), "bytes": int(nbytes), "GB_s": round(gbs, 1),
                                "frac_hbm": round(gbs / hbm, 3)}
    for sd, d in decode_roof.items():
        d["frac_hbm"] = round(d["GB_s"] / hbm, 3)
    value = S * world / (ms * 1e-3)
    line = {
        "metric": METRIC if args.workload == "c3" else f"MoE-layer fwd tokens/s @{args.workload}",
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": wl["desc"], "tokens_per_gpu": S, "global_batch": S * world,
                   "parallelism": f"ep{world}" if world > 1 else "single",
                   **({"transport": layer.transport, "schedule": layer.schedule,
                       "chunks": getattr(layer, "chunks", 1)}
                      if world > 1 else {}),
                   "l2": "inputs larger "
                   "than L2 (x 268 MB, expert weights 8.6 GB per layer)"},
        "roofline": {"bound": "tensor",
                     "kernel": "grouped expert GEMM (GEMM1+GEMM2" +
                               (" + shared-MLP GEMMs)" if residual else ")"),
                     "achieved": achieved, "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": achieved / tf_sus if achieved else None, "traffic": traffic,
                     "peak_kind": f"{src} sustained (burst {tf_burst})",
                     "frac_of_burst": achieved / tf_burst if achieved else None},
        "phases_ms": phases,
        "decode_p50_ms": decode or None,
        "decode_roofline": decode_roof or None,
        "components": components,
        "train_step": train,
        "kept_assignments_per_gpu": kept_rank,
        "cpu_baseline": cpu,
        "e2e": {"value": S * world / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": S * M * 2, "d2h_bytes_per_step": S * M * 2},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
