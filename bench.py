"""MoE-layer forward benchmark (BASELINE.json metric: tokens/s at the
1.3B+MoE-128 layer shape on 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step is one full MoE-layer forward (gate GEMM + routing epilogue, capacity
scan, dispatch, grouped expert GEMM1/GEMM2, combine + residual) over one batch
of synthetic tokens already resident in HBM. N=1 runs BASELINE config 3 on one
GPU (S=65536, d_model=2048, d_ff=8192, 128 experts, top-1, cf=1.0, bf16).
N>1 (torchrun, one rank per GPU, NCCL) runs the expert-parallel layer with
S=65536 tokens per rank (weak scaling: global batch 65536*N, global capacity).

``--impl reference`` times the reference's own CPU implementation: the
unmodified ``moekit`` package (installed into oracle/_ref by
``__graft_entry__.build()``; the oracle port oracle/moe_oracle.py stands in
when it is absent) on the host cores, on the same workload and config: the
full-batch routing every step, the per-expert loop on a rotating sample of
experts scaled to all of them (CpuLayerStep).

Timing: per-step CUDA events on the launching stream; ``ms_per_step`` is the
timed region / K (inputs larger than L2) or the mean step time with a read-only
L2 flush between steps (inputs that fit L2); ``p50_ms`` the median step. The
roofline divides by the burst bf16 peak when the timed region is under 1 s and
by the sustained one otherwise; ``sustained`` repeats the step for >= 2 s.
"""

from __future__ import annotations

import argparse
import dataclasses
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
    ap.add_argument("--no-cpu-legs", action="store_true",
                    help="reference arm: skip the C1 / C2 / C3 CPU legs")
    ap.add_argument("--sustained-s", type=float, default=2.0,
                    help="seconds of the power-capped steady-state loop (0: skip)")
    ap.add_argument("--l2-flush", default="auto", choices=["auto", "on", "off"],
                    help="read-only L2 flush between timed steps (auto: when x fits L2)")
    ap.add_argument("--drop-variant", action="store_true",
                    help="N=1: SURVEY 8(d)'s drop-exercising logits (~45%% dropped at C3)")
    ap.add_argument("--no-strong", action="store_true",
                    help="N>1: skip the C3 strong-scaling point (64K tokens in total)")
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
# CPU reference arm: the unmodified reference (moekit, installed under
# oracle/_ref by __graft_entry__.build()) on the host cores; the oracle port
# (oracle/moe_oracle.py) stands in only when that install is absent
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _reference_pkg():
    """moekit from oracle/_ref (kind "reference"), or None (kind "port")."""
    if not os.path.isdir(os.path.join(REF_DIR, "moekit")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import moekit.arch  # noqa: F401
    import moekit.gating  # noqa: F401
    import moekit.tensor  # noqa: F401

    return sys.modules["moekit"]


class CpuLayerStep:
    """One MoE-layer forward of a workload on the host CPU, float64 (the
    reference's only precision), as ``moekit.arch.forward_layer`` runs it
    (arch.py:372-413): the gate matmul, top_k_gate, build_dispatch_plan and
    row_softmax over the FULL batch, then the per-expert loop of
    ``_combine_experts`` (gather rows, forward_ffn, gate-prob scale, dense
    scatter_rows + accumulate), the residual add (+ the shared MLP).

    Bounded sample: every step times the full-batch routing and the reference's
    own ``_combine_experts`` on a rotating sample of ``n_sample`` experts (the
    plan restricted to them), then extrapolates the expert loop to every expert
    with kept rows: step = routing + skip-add + sampled_loop * active / n_sample.
    The per-expert body is identical for every expert (same row count up to the
    load, same FFN shape), so the extrapolation is per-expert cost x count."""

    def __init__(self, wl: dict, n_sample: int = 2, seed: int = 0) -> None:
        self.S, self.M, self.E, self.k, self.cf = wl["S"], wl["M"], wl["E"], wl["k"], wl["cf"]
        self.residual = wl["residual"]
        self.mk = _reference_pkg()
        self.kind = "reference" if self.mk is not None else "port"
        self.n_sample = min(n_sample, self.E)
        rng = np.random.default_rng(seed)
        M, F = self.M, 4 * self.M
        self.x = rng.standard_normal((self.S, M))
        self.gw = rng.standard_normal((M, self.E)) * 0.1

        def ffn():
            return (rng.standard_normal((M, F)) * 0.1, np.zeros((1, F)),
                    rng.standard_normal((F, M)) * 0.1, np.zeros((1, M)))

        # distinct weights per sampled slot (expert e uses pool[e % n]): the sampled
        # experts read their own weights, like the reference's per-expert params
        self.pool = [ffn() for _ in range(self.n_sample)]
        self.shared = ffn() if self.residual else None
        self.next = 0
        if self.mk is not None:
            A, G, T = self.mk.arch, self.mk.gating, self.mk.tensor
            self.cfg = G.GatingConfig(self.E, self.k, self.cf)
            self.xt = T.Tensor(self.x)
            self.gwt = T.Tensor(self.gw)
            wrap = lambda p: A.FfnParams(*(T.Tensor(a) for a in p))  # noqa: E731
            pool = [wrap(p) for p in self.pool]
            self.params = A.MoeLayerParams(gate_w=self.gwt,
                                           experts=tuple(pool[e % self.n_sample]
                                                         for e in range(self.E)),
                                           shared=wrap(self.shared) if self.residual else None)

    def desc(self) -> str:
        src = ("unmodified moekit (oracle/_ref) forward_layer pieces: tk.matmul gate, "
               "top_k_gate, build_dispatch_plan, row_softmax, arch._combine_experts"
               if self.kind == "reference" else "oracle port of forward_layer")
        return (f"{src}, float64, S={self.S} d_model={self.M} d_ff={4 * self.M} E={self.E} "
                f"k={self.k} cf={self.cf}{' + shared MLP' if self.residual else ''}: routing "
                f"and skip-add timed on the full batch every step, the expert loop timed on "
                f"{self.n_sample} rotating experts per step and scaled to every expert with "
                f"kept rows")

    def _sample(self, load: np.ndarray) -> list:
        active = [e for e in range(self.E) if load[e] > 0]
        if not active:
            return []
        out = []
        for _ in range(min(self.n_sample, len(active))):
            out.append(active[self.next % len(active)])
            self.next += 1
        return sorted(set(out))

    def step(self) -> tuple:
        """-> (extrapolated seconds for one full-layer forward, detail dict)."""
        t0 = time.perf_counter()
        if self.mk is not None:
            A, G, T = self.mk.arch, self.mk.gating, self.mk.tensor
            logits = T.matmul(self.xt, self.gwt)  # arch.py:384
            gates = G.top_k_gate(logits.value, self.cfg)
            plan = G.build_dispatch_plan(gates, self.cfg, self.S)
            probs = T.row_softmax(logits)
            load = plan.expert_load
            t1 = time.perf_counter()
            sample = self._sample(load)
            keep = np.isin(plan.expert_ids, sample)
            sub = dataclasses.replace(plan, slots=np.where(keep, plan.slots, G.DROPPED))
            acc = A._combine_experts(self.xt, probs, sub, self.params)  # arch.py:395-413
            t2 = time.perf_counter()
            out = T.add(self.xt, acc)  # arch.py:389
            if self.residual:
                out = T.add(out, A.forward_ffn(self.xt, self.params.shared))  # arch.py:390-391
        else:
            from oracle import moe_oracle as O

            logits = self.x @ self.gw
            ids, _, probs = O.top_k_gate(logits, self.E, self.k)
            slots, load, _ = O.build_dispatch_plan(ids, self.E, self.k, self.cf)
            t1 = time.perf_counter()
            sample = self._sample(load)
            acc = np.zeros_like(self.x)
            for e in sample:
                sel = (slots != -1) & (ids == e)
                rows = np.nonzero(sel.any(axis=1))[0]
                rows = rows[np.argsort(slots[sel], kind="stable")]
                y = O.forward_ffn(self.x[rows], *self.pool[e % self.n_sample])
                contrib = np.zeros_like(self.x)
                contrib[rows] = y * probs[rows, e][:, None]
                acc = acc + contrib
            t2 = time.perf_counter()
            out = self.x + acc
            if self.residual:
                out = out + O.forward_ffn(self.x, *self.shared)
        t3 = time.perf_counter()
        active = int((np.asarray(load) > 0).sum())
        loop = (t2 - t1) * (active / len(sample)) if sample else 0.0
        est = (t1 - t0) + (t3 - t2) + loop
        return est, {"routing_s": t1 - t0, "skip_add_s": t3 - t2, "sampled_loop_s": t2 - t1,
                     "sampled_experts": len(sample), "active_experts": active}


def _blas_threads(n: int | None = None) -> int:
    """Set the BLAS pool (torchrun exports OMP_NUM_THREADS=1, which OpenBLAS read
    at import; threadpoolctl changes it at run time). n=None: every host core."""
    cores = n or len(os.sched_getaffinity(0))
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=cores)
    except Exception:  # noqa: BLE001 - keep whatever the BLAS was started with
        pass
    return cores


def cpu_baseline_sample(wl: dict, steps: int = 2) -> dict:
    """The GPU arm's cpu_baseline: the CPU layer step, one warm-up + ``steps``."""
    cores = _blas_threads()
    c = CpuLayerStep(wl)
    c.step()
    est = [c.step()[0] for _ in range(steps)]
    v = wl["S"] / statistics.median(est)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": c.kind,
            "sample": c.desc() + f"; median of {steps} steps after one warm-up, "
                                 f"{cores} BLAS threads"}


def _median_time(fn, reps: int) -> float:
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def cpu_reference_legs(mk) -> dict:
    """SURVEY 8(d)'s other CPU legs, on the unmodified reference: forward_layer at
    C1 (all cores and 1 thread), and routing only - top_k_gate,
    build_dispatch_plan, scatter_tokens, combine_tokens - over the full C2 and
    C3 batches. Median of 3 after one warm-up each."""
    from threadpoolctl import threadpool_limits

    A, G, T = mk.arch, mk.gating, mk.tensor
    legs = {}
    rng = np.random.default_rng(0)
    spec = A.LayerSpec(kind="moe", hidden=1024, experts=8, gating=G.GatingConfig(8, 1, 1.0))
    params = A.init_layer_params(spec, rng)
    x = T.Tensor(rng.standard_normal((4096, 1024)))
    run = lambda: A.forward_layer(x, spec, params)  # noqa: E731
    t_all = _median_time(run, 3)
    with threadpool_limits(limits=1):
        t_one = _median_time(run, 2)
    legs["c1_forward_layer"] = {"tokens": 4096, "s_all_cores": t_all, "s_1_thread": t_one,
                               "tokens_per_s_all_cores": 4096 / t_all,
                               "tokens_per_s_1_thread": 4096 / t_one}
    for name, (S, M, E, k, cf) in (("c2_routing", (16384, 1024, 16, 2, 1.25)),
                                   ("c3_routing", (65536, 2048, 128, 1, 1.0))):
        cfg = G.GatingConfig(E, k, cf)
        lg = rng.standard_normal((S, E))
        xb = rng.standard_normal((S, M))
        parts = {}

        def route():
            t0 = time.perf_counter()
            g = G.top_k_gate(lg, cfg)
            t1 = time.perf_counter()
            plan = G.build_dispatch_plan(g, cfg, S)
            t2 = time.perf_counter()
            buf = G.scatter_tokens(xb, plan)
            t3 = time.perf_counter()
            G.combine_tokens(buf, plan)
            t4 = time.perf_counter()
            for kk, v in zip(("top_k_gate", "build_dispatch_plan", "scatter_tokens",
                              "combine_tokens"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
                parts.setdefault(kk, []).append(v)

        tot = _median_time(route, 3)
        legs[name] = {"tokens": S, "s": tot, "tokens_per_s": S / tot,
                      **{kk + "_s": statistics.median(v[1:]) for kk, v in parts.items()}}
    return legs


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    cores = _blas_threads()
    c = CpuLayerStep(wl)
    t_start = time.time()
    for _ in range(args.warmup):
        c.step()
    ests, details = [], []
    # every step is a few seconds of CPU work: the timed steps stop after ~120 s so
    # the arm ends within a few minutes whatever --steps is (the line reports both)
    for _ in range(args.steps):
        est, det = c.step()
        ests.append(est)
        details.append(det)
        if time.time() - t_start > 120.0:
            break
    med = statistics.median(ests)
    value = wl["S"] / med
    # one step on a single BLAS thread, one sampled expert (the 1-thread figure)
    one = None
    try:
        from threadpoolctl import threadpool_limits

        with threadpool_limits(limits=1):
            c1 = CpuLayerStep(wl, n_sample=1, seed=1)
            one = wl["S"] / c1.step()[0]
    except Exception as e:  # noqa: BLE001
        one = f"unavailable: {e}"
    legs = None
    if c.mk is not None and args.workload == "c3" and not args.no_cpu_legs:
        legs = cpu_reference_legs(c.mk)
    mean = lambda kk: statistics.mean(d[kk] for d in details)  # noqa: E731
    line = {
        "impl": "reference", "metric": metric_name(args.workload), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(ests), "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": med * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.workload, wl["S"], args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": c.kind,
                         "sample": c.desc(), "value_1_thread": one,
                         "per_step_mean_s": {kk: mean(kk) for kk in ("routing_s", "skip_add_s",
                                                                    "sampled_loop_s")},
                         "sampled_experts_per_step": details[0]["sampled_experts"],
                         "active_experts": details[0]["active_experts"]},
        "cpu_legs": legs,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampler (every 25 ms), started before the warm-up so it is up
    when a timed region begins; ``window(t0, t1)`` summarises the samples
    stamped inside one timed region (several windows per run)."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        self.idx = gpu_index
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "25"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def _samples(self) -> list:
        import datetime

        self.f.flush()
        stamped = []
        for line in open(self.f.name):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                stamped.append((ts, (float(parts[1]), float(parts[2]), float(parts[3]),
                                     parts[5:9])))
            except ValueError:
                continue
        return stamped

    def window(self, t0: float, t1: float) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)  # let the sampler flush the last rows of the window
        stamped = self._samples()
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
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v == "Active"})
        out = {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": mx,
               "power_w_median": statistics.median(r[2] for r in loaded),
               "reasons": reasons, "samples": len(rows)}
        if note:
            out["note"] = note
        return out

    def close(self) -> None:
        if self.p is not None:
            self.p.terminate()
            self.p.wait()
        try:
            os.unlink(self.f.name)
        except OSError:
            pass


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def make_layer(S, M, E, k, cf, dev, seed=0, residual=False, drop_variant=False):
    import torch

    from paper_2201_05596_b200 import arch as A
    from paper_2201_05596_b200.gating import GatingConfig

    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=residual,
                       gating=GatingConfig(E, k, cf))
    gen = torch.Generator(device=dev).manual_seed(seed)
    F = 4 * M
    # random-init weights of the named architecture: N(0,1)*0.1, zero biases (arch.py:347-365)
    gw = torch.randn(M, E, device=dev, generator=gen) * 0.1
    if drop_variant:
        # SURVEY 8(d) drop-exercising variant: unit-scale logits plus a per-expert
        # bias N(0, 0.5^2), entering through the constant input feature x[:, 0] = 1
        gw = torch.randn(M, E, device=dev, generator=gen) * M ** -0.5
        gw[0] = torch.randn(E, device=dev, generator=gen) * 0.5
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


L2_BYTES = 126 * 2 ** 20


def metric_name(workload: str) -> str:
    return METRIC if workload == "c3" else f"MoE-layer fwd tokens/s @{workload}"


def bench_config(workload: str, S: int, world: int) -> dict:
    """The line's config (identical in both arms, so the driver can pair them)."""
    wl = WORKLOADS[workload]
    return {"workload": wl["desc"], "tokens_per_gpu": S, "global_batch": S * world,
            "parallelism": f"ep{world}" if world > 1 else "single"}


def l2_policy(S: int, M: int, E: int, residual: bool) -> tuple:
    """-> (flush between steps?, note). Inputs larger than L2 need no flush; a
    batch that fits (C2 / C4: x 34 MB) is evicted by a read-only flush between
    timed steps (the flush is outside each step's event pair)."""
    xb = S * M * 2
    wb = E * 2 * M * 4 * M * 2 + (2 * M * 4 * M * 2 if residual else 0)
    if xb > L2_BYTES:
        return False, (f"inputs larger than L2 (x {xb / 1e6:.0f} MB, expert weights "
                       f"{wb / 1e9:.2f} GB vs 126 MB L2): steps back to back, no flush")
    return True, (f"x {xb / 1e6:.0f} MB fits the 126 MB L2 (expert weights {wb / 1e9:.2f} GB "
                  f"do not): a 512 MB read-only L2 flush runs between timed steps, outside "
                  f"each step's event pair; ms_per_step = mean of the per-step times")


def timed_steps(layer, x, out, steps, flush_buf=None, timer=None):
    """K forwards; per-step CUDA events on the launching stream. Returns
    (per-step ms list, total ms of the region, whether steps ran back to back)."""
    import torch

    if flush_buf is None:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record()
        for i in range(steps):
            layer(x, out=out, timer=timer)
            ev[i + 1].record()
        torch.cuda.synchronize()
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
        return per, ev[0].elapsed_time(ev[-1])
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record()
    for i in range(steps):
        torch.amax(flush_buf)  # read-only: evicts x without leaving dirty lines
        e0[i].record()
        layer(x, out=out, timer=timer)
        e1[i].record()
    g1.record()
    torch.cuda.synchronize()
    per = [e0[i].elapsed_time(e1[i]) for i in range(steps)]
    return per, g0.elapsed_time(g1)


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
        # NCCL's own banner (NCCL_DEBUG=VERSION prints it on stdout when the first
        # communicator comes up) goes to stderr: rank 0's stdout carries one JSON line
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()
            torch.cuda.synchronize()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
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
        layer = make_layer(S, M, E, k, cf, dev, residual=residual, drop_variant=args.drop_variant)
    gen = torch.Generator(device=dev).manual_seed(1 + rank)
    x = torch.randn(S, M, device=dev, generator=gen).to(torch.bfloat16)
    if args.drop_variant:
        x[:, 0] = 1.0
    # synthetic routing with unbiased logits: ~4% drops at C3
    # (expert-parallel layers return their own output: for k=1 layers the owners'
    # GEMM2 epilogues store the combined rows straight into it over NVLink)
    out = torch.empty_like(x) if world == 1 else None
    flush, l2_note = l2_policy(S, M, E, residual)
    if args.l2_flush != "auto":  # diagnostic override (e.g. gate timing after a clean L2)
        flush = args.l2_flush == "on"
        l2_note += f"; overridden: flush {'on' if flush else 'off'}"
    flush_buf = torch.empty(512 * 2 ** 20 // 2, dtype=torch.float16, device=dev).fill_(0) \
        if flush else None
    clocks = Clocks(local) if rank == 0 else None
    for _ in range(args.warmup):
        layer(x, out=out)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: K full forwards, inputs resident in HBM
    timer = _lib.PhaseTimer()
    launches0 = _lib.launch_count()
    barrier()
    w0 = time.time()
    per, region_ms = timed_steps(layer, x, out, args.steps, flush_buf, timer)
    w1 = time.time()
    barrier()
    launches = _lib.launch_count() - launches0
    if hasattr(layer, "check_errors"):
        layer.check_errors()  # a timed-out peer barrier fails the run loudly
    clk = clocks.window(w0, w1) if clocks else None
    ms = max_over_ranks(statistics.mean(per) if flush else region_ms / args.steps)
    p50 = max_over_ranks(statistics.median(per))
    region_ms = max_over_ranks(region_ms)
    phases = timer.summary(args.steps)
    kept = int(layer.kept_assignments(S)) if hasattr(layer, "kept_assignments") else S * k
    hbm, tf_burst, tf_sus, src = peaks()

    def gemm_ms_of(ph: dict) -> float:
        return sum(v for kk, v in ph.items() if kk.startswith("gemm") or kk.startswith("shared_mlp"))

    # ---- sustained: the same step looped for >= 2 s (the timed region above is a
    # short burst at full clock; this is the 1 kW power-capped steady state)
    sustained = None
    if args.sustained_s > 0:
        n_sus = max(int(args.sustained_s * 1e3 / max(ms, 1e-3)) + 1, args.steps)
        t_sus = _lib.PhaseTimer()
        barrier()
        s0 = time.time()
        per_s, reg_s = timed_steps(layer, x, out, n_sus, flush_buf, t_sus)
        s1 = time.time()
        barrier()
        ms_s = max_over_ranks(statistics.mean(per_s) if flush else reg_s / n_sus)
        ph_s = t_sus.summary(n_sus)
        sustained = {"steps": n_sus, "seconds": round(max_over_ranks(reg_s) / 1e3, 3),
                     "ms_per_step": ms_s, "p50_ms": max_over_ranks(statistics.median(per_s)),
                     "tokens_per_s": S * world / (ms_s * 1e-3),
                     "gemm_ms": gemm_ms_of(ph_s),
                     "clocks": clocks.window(s0, s1) if clocks else None}
    # ---- C3 strong-scaling point at N>1 (BASELINE config 3: 64K tokens in total,
    # split over the N GPUs) beside the weak-scaling headline
    strong = None
    if world > 1 and args.workload == "c3" and not args.no_strong:
        s_loc = 65536 // world
        xs = x[:s_loc].contiguous()
        os_ = None
        for _ in range(3):
            layer(xs, out=os_)
        barrier()
        per_st, reg_st = timed_steps(layer, xs, os_, args.steps)
        barrier()
        ms_st = max_over_ranks(reg_st / args.steps)
        strong = {"global_batch": 65536, "tokens_per_gpu": s_loc, "ms_per_step": ms_st,
                  "p50_ms": max_over_ranks(statistics.median(per_st)),
                  "tokens_per_s": 65536 / (ms_st * 1e-3), "scaling": "strong"}
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
        per_t = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.train_steps)]
        tms = ev[0].elapsed_time(ev[-1]) / args.train_steps
        train = {"ms_per_step": round(tms, 3), "ms_per_step_median": round(statistics.median(per_t), 3),
                 "tokens_per_s": S / (tms * 1e-3),
                 "gemm_tflops": 12.0 * kept * M * F / (tms * 1e-3) / 1e12,
                 "steps": args.train_steps, "note": "forward_train + backward, bf16"}
        layer._train_ctx = None
        torch.cuda.empty_cache()
    # ---- e2e through the public API: pinned host x -> layer(x) -> pinned host out.
    # Each step uploads its batch and downloads its result; the layer streams host
    # batches (H2D / forward / D2H overlapped across steps).
    xh = x.cpu().pin_memory()
    ohs = [torch.empty_like(xh).pin_memory() for _ in range(2)]
    for i in range(2):
        layer(xh, out=ohs[i % 2])
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        layer(xh, out=ohs[i % 2])
    layer._pipe.wait()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    if world > 1:
        kt = torch.tensor([kept], device=dev, dtype=torch.int64)
        dist.all_reduce(kt)
        kept_total = int(kt.item())
    else:
        kept_total = kept
    if clocks:
        clocks.close()

    if rank != 0:
        dist.destroy_process_group()
        return
    # dominant kernel: the grouped expert GEMM (GEMM1 + GEMM2 launches); the peak is
    # the burst one for a short timed region, the sustained one for >= 1 s
    gemm_ms = gemm_ms_of(phases)
    kept_rank = kept_total / world
    # 2*A*M*F per expert GEMM launch (two launches), + 4*S*M*F for the shared MLP
    flops_step = 4.0 * kept_rank * M * F + (4.0 * S * M * F if residual else 0.0)
    achieved = flops_step / (gemm_ms * 1e-3) / 1e12 if gemm_ms else None
    short = region_ms < 1000.0
    peak = tf_burst if short else tf_sus
    roof = {"bound": "tensor",
            "kernel": "grouped expert GEMM (GEMM1+GEMM2" +
                      (" + shared-MLP GEMMs)" if residual else ")"),
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if achieved else None,
            "traffic": measured_traffic(args.workload, world),
            "peak_kind": (f"{src} burst bf16 (timed region {region_ms:.0f} ms < 1 s)" if short
                          else f"{src} sustained bf16 (timed region {region_ms / 1e3:.1f} s)"),
            "algorithmic_flops_per_step": flops_step,
            "flops_formula": "4*A*M*F (+4*S*M*F shared MLP), A = kept assignments per GPU"}
    if sustained:
        a_s = flops_step / (sustained["gemm_ms"] * 1e-3) / 1e12 if sustained["gemm_ms"] else None
        sustained["gemm_tflops"] = a_s
        sustained["gemm_frac_of_sustained_peak"] = a_s / tf_sus if a_s else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(wl)
    # HBM-bound components (SURVEY 8(d) formulas, per rank, phase times from the
    # timed region): achieved GB/s and fraction of the measured HBM peak
    A_r = kept_rank
    T_r = (S + 127) // 128
    epad = max(32, 1 << (E - 1).bit_length())
    # dispatch: kept rows read + written; the k=1 fused dispatch also copies every
    # fully dropped token to out (its skip connection), so it moves every row once
    fused_k1 = world == 1 and k == 1 and not residual
    comp_bytes = {"gate": S * M * 2 + epad * M * 2 + S * k * 12 + T_r * E * 4,
                  "dispatch": (2 * S * M * 2) if fused_k1 else 2 * A_r * M * 2,
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
    cfg = bench_config(args.workload, S, world)  # identical dict in the reference arm
    ep_cfg = ({"transport": layer.transport, "schedule": layer.schedule,
               "chunks": getattr(layer, "chunks", 1)} if world > 1 else None)
    line = {
        "metric": metric_name(args.workload),
        "value": S * world / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "p50_ms": p50,
        "step_ms": {"min": min(per), "max": max(per), "first": per[0],
                    "all": [round(v, 4) for v in per] if len(per) <= 50 else None},
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": cfg, "ep": ep_cfg, "l2": l2_note,
        "roofline": roof,
        "sustained": sustained,
        "strong_scaling": strong,
        "phases_ms": phases,
        "decode_p50_ms": decode or None,
        "decode_roofline": decode_roof or None,
        "components": components,
        "train_step": train,
        "kept_assignments_per_gpu": kept_rank,
        "drop_variant": bool(args.drop_variant),
        "cpu_baseline": cpu,
        "e2e": {"value": S * world / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": S * M * 2, "d2h_bytes_per_step": S * M * 2},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measured_traffic(workload: str, world: int):
    """DRAM bytes (read + write) of the grouped-GEMM launches of one step, from an
    ncu capture of THIS workload (profiles/traffic.json, keyed by workload and
    GPU count), or None when no capture of it exists."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    t = json.load(open(path)).get(f"{workload}_n{world}")
    return None if t is None else t.get("grouped_gemm_bytes_per_step")


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
