"""Generate golden vectors by running the REFERENCE package (moekit) itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Writes small .npz fixtures next to this script. They pin the oracle
(oracle/moe_oracle.py) and the GPU path to the reference's own outputs. The
cases mirror the reference test suite (pkg/tests/test_gating.py,
pkg/tests/test_arch.py::TestForward, pkg/tests/test_acceptance.py C4/C5/C8).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

from moekit import gating  # noqa: E402
from moekit import tensor as tk  # noqa: E402
from moekit.arch import LayerSpec, forward_ffn, forward_layer, init_layer_params, load_balance_loss  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in arrays.values()), "bytes raw")


def gate_kats():
    # test_gating.py:65-98 plus the survey's extra tie cases
    cases = [
        ([[1.0, 3.0, 2.0]], 1),
        ([[1.0, 3.0, 2.0]], 2),
        ([[5.0, 5.0, 1.0]], 2),
        ([[2.0, 7.0, 7.0, 7.0]], 1),
        ([[0.4, 2.0, -1.0, 1.5]], 2),
        ([[0.0, -0.0, 1.0, 1.0]], 2),
        ([[3.0, 3.0, 3.0, 3.0]], 2),
        ([[-1.0, -2.0]], 2),
    ]
    out = {}
    for i, (logits, k) in enumerate(cases):
        lg = np.array(logits)
        cfg = gating.GatingConfig(num_experts=lg.shape[1], k=k)
        g = gating.top_k_gate(lg, cfg)
        out[f"c{i}_logits"] = lg
        out[f"c{i}_k"] = np.array(k)
        out[f"c{i}_ids"] = g.expert_ids
        out[f"c{i}_gp"] = g.gate_probs
        out[f"c{i}_probs"] = g.probs
    # random rows with forced ties (fp32-representable values)
    rng = np.random.default_rng(42)
    for i in range(8, 14):
        s, e = int(rng.integers(1, 200)), int(rng.integers(2, 129))
        k = int(rng.integers(1, 3))
        lg = rng.integers(-3, 4, size=(s, e)).astype(np.float64) * 0.5
        cfg = gating.GatingConfig(num_experts=e, k=k)
        g = gating.top_k_gate(lg, cfg)
        out[f"c{i}_logits"] = lg
        out[f"c{i}_k"] = np.array(k)
        out[f"c{i}_ids"] = g.expert_ids
        out[f"c{i}_gp"] = g.gate_probs
        out[f"c{i}_probs"] = g.probs
    out["n"] = np.array(14)
    _save("gate_kats.npz", **out)


def scans():
    # test_gating.py:121-150, test_acceptance.py:168-187
    rng = np.random.default_rng(1)
    out = {"worked_in": np.array([3, 1, 7, 0, 4, 1, 6, 3]),
           "worked_out": gating.exclusive_scan_blelloch(np.array([3, 1, 7, 0, 4, 1, 6, 3]))}
    lengths = list(range(0, 70)) + [127, 128, 129, 255, 256, 257, 1023, 1024, 1025, 4097, 50000]
    for i, n in enumerate(lengths):
        v = rng.integers(0, 10, size=n)
        out[f"i{i}_in"] = v
        out[f"i{i}_out"] = gating.exclusive_scan_blelloch(v)
    # float input: float64 result in tree order
    for i, n in enumerate([1, 5, 8, 33, 1000, 4099]):
        v = rng.standard_normal(n)
        out[f"f{i}_in"] = v
        out[f"f{i}_out"] = gating.exclusive_scan_blelloch(v)
    out["n_int"] = np.array(len(lengths))
    out["n_float"] = np.array(6)
    _save("scans.npz", **out)


def plans():
    # test_gating.py:158-249 KATs + 40 random trials vs brute force (:193-206)
    out = {}
    cases = []
    cases.append((np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 0.0]]), 1, 1.0))
    lg = np.zeros((8, 4)); lg[:, 0] = 5.0
    cases.append((lg, 1, 0.5))
    cases.append((np.array([[2.0, 1.0], [3.0, 0.0]]), 2, 1.0))
    cases.append((np.zeros((0, 4)), 1, 1.0))
    rng = np.random.default_rng(3)
    for _ in range(40):
        s = int(rng.integers(1, 65)); e = int(rng.integers(2, 9))
        k = int(rng.choice([1, 2])); cf = float(rng.choice([0.5, 1.0, 2.0]))
        cases.append((rng.standard_normal((s, e)), k, cf))
    # larger, skewed (drop-exercising) instances
    rng = np.random.default_rng(33)
    for s, e, k, cf in [(4096, 16, 2, 1.25), (2048, 128, 1, 1.0), (3000, 64, 2, 0.5), (1000, 7, 1, 1.5)]:
        lg = rng.standard_normal((s, e)) + rng.normal(0, 0.5, size=(1, e))
        cases.append((lg.astype(np.float32).astype(np.float64), k, cf))
    for i, (lg, k, cf) in enumerate(cases):
        cfg = gating.GatingConfig(num_experts=lg.shape[1], k=k, capacity_factor=cf)
        g = gating.top_k_gate(lg, cfg)
        p = gating.build_dispatch_plan(g, cfg, lg.shape[0])
        out[f"p{i}_logits"] = lg
        out[f"p{i}_cfg"] = np.array([lg.shape[1], k, cf])
        out[f"p{i}_ids"] = p.expert_ids
        out[f"p{i}_gp"] = p.gate_probs
        out[f"p{i}_slots"] = p.slots
        out[f"p{i}_load"] = p.expert_load
        out[f"p{i}_cap"] = np.array(p.capacity)
        out[f"p{i}_lbl"] = np.array(load_balance_loss(p, g.probs))
    out["n"] = np.array(len(cases))
    caps = []
    for e, k, cf, s in [(64, 1, 1.0, 512), (64, 1, 1.25, 512), (64, 2, 1.0, 512), (4, 1, 1e-9, 8),
                        (4, 1, 1.0, 0), (128, 1, 1.0, 65536), (16, 2, 1.25, 16384), (128, 1, 1.0, 64),
                        (8, 1, 1.0, 4096), (32, 1, 1.0, 16384), (64, 1, 1.0, 16384), (3, 2, 0.7, 1001)]:
        caps.append([e, k, cf, s, gating.GatingConfig(e, k, cf).capacity(s)])
    out["capacity_table"] = np.array(caps, dtype=np.float64)
    _save("plans.npz", **out)


def scatter_combine():
    # test_gating.py:270-348 random instances; acceptance C4 shape range
    rng = np.random.default_rng(2024)
    out = {}
    n = 30
    for i in range(n):
        s = int(rng.integers(1, 257)); e = int(rng.integers(1, 17))
        k = int(rng.integers(1, 3)) if e >= 2 else 1
        cf = float(rng.choice([0.5, 1.0, 2.0])); m = int(rng.integers(1, 40))
        cfg = gating.GatingConfig(num_experts=e, k=k, capacity_factor=cf)
        g = gating.top_k_gate(rng.standard_normal((s, e)), cfg)
        p = gating.build_dispatch_plan(g, cfg, s)
        x = rng.standard_normal((s, m))
        counter = gating.OpCounter()
        buf = gating.scatter_tokens(x, p, counter)
        y = np.tanh(buf.data)

        class _B:
            data = y
            occupied = buf.occupied
        comb = gating.combine_tokens(_B, p, counter)
        out[f"s{i}_x"] = x
        out[f"s{i}_cfg"] = np.array([e, k, cf])
        out[f"s{i}_ids"] = p.expert_ids
        out[f"s{i}_gp"] = p.gate_probs
        out[f"s{i}_slots"] = p.slots
        out[f"s{i}_data"] = buf.data
        out[f"s{i}_occ"] = buf.occupied
        out[f"s{i}_comb"] = comb
        out[f"s{i}_ops"] = np.array(counter.ops)
    out["n"] = np.array(n)
    _save("scatter_combine.npz", **out)


def layers():
    # test_arch.py:222-296 + acceptance C8 + survey S=257,E=8,M=16
    out = {}
    cases = [
        (257, 16, 8, 1, 1.0, False, 0),
        (257, 16, 8, 2, 1.0, False, 1),
        (257, 16, 8, 1, 1.0, True, 2),
        (257, 16, 8, 2, 1.25, True, 3),
        (6, 8, 2, 1, 1e-9, False, 24),     # dropped tokens ride the skip (test_arch.py:267-275)
        (12, 32, 1, 1, 16.0, False, 1),    # single expert == dense (C8)
        (64, 24, 4, 2, 0.5, False, 7),
        (100, 12, 16, 1, 1.0, True, 9),
    ]
    for i, (s, m, e, k, cf, res, seed) in enumerate(cases):
        spec = LayerSpec(kind="moe", hidden=m, experts=e, residual=res,
                         gating=gating.GatingConfig(num_experts=e, k=k, capacity_factor=cf))
        rng = np.random.default_rng(seed)
        params = init_layer_params(spec, rng)
        # non-zero biases so bias plumbing is exercised
        for f in list(params.experts) + ([params.shared] if params.shared else []):
            f.b1.value[:] = rng.standard_normal(f.b1.value.shape) * 0.05
            f.b2.value[:] = rng.standard_normal(f.b2.value.shape) * 0.05
        x = rng.standard_normal((s, m))
        y = forward_layer(tk.Tensor(x), spec, params).value
        out[f"l{i}_cfg"] = np.array([s, m, e, k, cf, float(res)])
        out[f"l{i}_x"] = x
        out[f"l{i}_gate_w"] = params.gate_w.value
        out[f"l{i}_w1"] = np.stack([f.w1.value for f in params.experts])
        out[f"l{i}_b1"] = np.stack([f.b1.value for f in params.experts])
        out[f"l{i}_w2"] = np.stack([f.w2.value for f in params.experts])
        out[f"l{i}_b2"] = np.stack([f.b2.value for f in params.experts])
        if res:
            sh = params.shared
            out[f"l{i}_sw1"], out[f"l{i}_sb1"] = sh.w1.value, sh.b1.value
            out[f"l{i}_sw2"], out[f"l{i}_sb2"] = sh.w2.value, sh.b2.value
            out[f"l{i}_shared_out"] = forward_ffn(tk.Tensor(x), sh).value
        out[f"l{i}_out"] = y
    out["n"] = np.array(len(cases))
    _save("layers.npz", **out)


def route_bench():
    # the reference CLI's route-bench verb (cli.py:260-306) on two configs
    import json
    import tempfile

    from moekit.cli import main

    for name, opts, seed in [("route_bench_a.csv", {"tokens": 300, "experts": 8, "k": 2,
                                                     "capacity_factor": 1.0, "instances": 5}, 7),
                             ("route_bench_b.csv", {"tokens": 1000, "experts": 16, "k": 1,
                                                     "capacity_factor": 0.5, "instances": 3}, 11)]:
        with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
            json.dump({"seed": seed, "options": opts}, f)
        rc = main(["route-bench", "--config", f.name, "--out", os.path.join(HERE, name)])
        assert rc == 0
        print("wrote", name)


def layer_grads():
    """Reference tape backward of loss = sum(forward_layer(x) * G) (arch.py:372-413,
    tensor.py GradTape): gradients w.r.t. x, gate_w, every expert's w1/b1/w2/b2 and
    the shared MLP. Inputs are bf16-representable so a bf16 device path sees them
    exactly."""
    from moekit.tensor import GradTape, Tensor, mul, sum_all

    def bf(a):
        a = np.asarray(a, dtype=np.float32)
        u = a.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000  # round-to-nearest-even to bf16
        return u.astype(np.uint32).view(np.float32).astype(np.float64)

    out = {}
    cases = [(256, 64, 8, 1, 1.0, False, 1), (256, 64, 8, 2, 1.25, True, 2),
             (200, 32, 4, 2, 0.6, False, 3), (300, 64, 8, 1, 0.5, True, 4)]
    for i, (s, m, e, k, cf, res, seed) in enumerate(cases):
        spec = LayerSpec(kind="moe", hidden=m, experts=e, residual=res,
                         gating=gating.GatingConfig(num_experts=e, k=k, capacity_factor=cf))
        rng = np.random.default_rng(100 + seed)
        params = init_layer_params(spec, rng)
        ffns = list(params.experts) + ([params.shared] if params.shared else [])
        params.gate_w.value[:] = bf(params.gate_w.value)
        for f in ffns:
            f.w1.value[:] = bf(f.w1.value)
            f.w2.value[:] = bf(f.w2.value)
            f.b1.value[:] = np.float32(rng.standard_normal(f.b1.value.shape) * 0.05)
            f.b2.value[:] = np.float32(rng.standard_normal(f.b2.value.shape) * 0.05)
        x = bf(rng.standard_normal((s, m)))
        g = bf(rng.standard_normal((s, m)))  # bf16-exact so every consumer sees it exactly
        tape = GradTape()
        xt = Tensor(x, tape)
        y = forward_layer(xt, spec, params)
        tape.backward(sum_all(mul(y, Tensor(g))))
        out[f"g{i}_cfg"] = np.array([s, m, e, k, cf, float(res)])
        out[f"g{i}_x"] = x
        out[f"g{i}_G"] = g
        out[f"g{i}_out"] = y.value
        out[f"g{i}_gate_w"] = params.gate_w.value
        out[f"g{i}_dx"] = xt.grad
        out[f"g{i}_dgate_w"] = params.gate_w.grad
        for n in ("w1", "b1", "w2", "b2"):
            out[f"g{i}_{n}"] = np.stack([getattr(f, n).value for f in params.experts])
            out[f"g{i}_d{n}"] = np.stack([
                getattr(f, n).grad if getattr(f, n).grad is not None
                else np.zeros_like(getattr(f, n).value) for f in params.experts])
            if res:
                sh = params.shared
                out[f"g{i}_s{n}"] = getattr(sh, n).value
                out[f"g{i}_ds{n}"] = getattr(sh, n).grad
    out["n"] = np.array(len(cases))
    # float32 is exact for the bf16 inputs and ample for bf16-tolerance gradients
    out = {kk: (v.astype(np.float32) if v.dtype == np.float64 and not kk.endswith("_cfg") else v)
           for kk, v in out.items()}
    _save("layer_grads.npz", **out)


def commsim_cases():
    """The reference's exchange schedules (commsim.py:239-464) on seeded payloads:
    per-rank send lists and the delivered receive lists, plus the trace totals."""
    from moekit import commsim as cs

    out = {}
    cases = []
    # (kind, world, param, per_rank, seed): param = gpus_per_node or tensor_slice
    for seed in range(3):
        cases.append(("hierarchical", 4, 2, 6, seed))
    cases.append(("hierarchical", 4, 4, 5, 7))
    cases.append(("hierarchical", 4, 1, 5, 8))
    cases.append(("hierarchical", 2, 2, 9, 9))
    for seed in range(3):
        cases.append(("coordinated", 4, 2, 7, 10 + seed))
    cases.append(("coordinated", 4, 4, 6, 20))
    cases.append(("coordinated", 4, 1, 6, 21))
    cases.append(("coordinated", 2, 2, 6, 22))
    for i, (kind, world, param, per, seed) in enumerate(cases):
        if kind == "hierarchical":
            sends = cs.synthetic_sends(world, per, nbytes=64, seed=seed)
            trace = cs.hierarchical_all_to_all(sends, param)
            flat = cs.flat_all_to_all(sends)
            assert trace.recv == flat.recv
            out[f"c{i}_flat_volume"] = np.array(flat.volume_bytes)
            out[f"c{i}_flat_rounds"] = np.array(flat.a2a_rounds)
        else:
            logical = cs.synthetic_sends(world // param, per, nbytes=64, seed=seed)
            sends = [list(items) for items in logical for _ in range(param)]
            trace = cs.coordinated_all_to_all(sends, param)
        out[f"c{i}_cfg"] = np.array([0 if kind == "hierarchical" else 1, world, param])
        out[f"c{i}_sends"] = np.array([[it.src, it.dst, it.token, it.nbytes]
                                       for items in sends for it in items], dtype=np.int64)
        out[f"c{i}_send_rank"] = np.array([r for r, items in enumerate(sends) for _ in items])
        out[f"c{i}_recv"] = np.array([[r, it.src, it.token] for r, items in enumerate(trace.recv)
                                      for it in items], dtype=np.int64).reshape(-1, 3)
        out[f"c{i}_stats"] = np.array([trace.a2a_rounds, trace.allgather_rounds,
                                       trace.volume_bytes, trace.a2a_volume_bytes,
                                       trace.reference_bytes], dtype=np.int64)
    out["n"] = np.array(len(cases))
    _save("commsim.npz", **out)


if __name__ == "__main__":
    commsim_cases()
    layer_grads()
    route_bench()
    gate_kats()
    scans()
    plans()
    scatter_combine()
    layers()
