"""GPU parity of the routing kernels against the reference's golden vectors and
the CPU oracle. Integer outputs (ids, slots, loads, scans) must be bit-exact;
float64 scatter/combine are bit-exact too (exact copies, individually rounded
IEEE ops); float64 softmax probabilities agree to a few ulp."""

import os

import numpy as np
import pytest
import torch

from oracle import moe_oracle as O
from paper_2201_05596_b200 import gating as G
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _load(name):
    return np.load(os.path.join(GOLDEN, name))


def test_gate_kats_golden():
    z = _load("gate_kats.npz")
    for i in range(int(z["n"])):
        lg, k = z[f"c{i}_logits"], int(z[f"c{i}_k"])
        g = G.top_k_gate(lg, G.GatingConfig(lg.shape[1], k))
        assert g.expert_ids.dtype == np.int64
        assert np.array_equal(g.expert_ids, z[f"c{i}_ids"]), i
        np.testing.assert_allclose(g.gate_probs, z[f"c{i}_gp"], rtol=1e-14, atol=1e-300)
        np.testing.assert_allclose(g.probs, z[f"c{i}_probs"], rtol=1e-14, atol=1e-300)


def test_gate_literal_kats():
    # test_gating.py:65-98
    assert G.top_k_gate(np.array([[1.0, 3.0, 2.0]]), G.GatingConfig(3, 1)).expert_ids.tolist() == [[1]]
    assert G.top_k_gate(np.array([[5.0, 5.0, 1.0]]), G.GatingConfig(3, 2)).expert_ids.tolist() == [[0, 1]]
    assert G.top_k_gate(np.array([[2.0, 7.0, 7.0, 7.0]]), G.GatingConfig(4, 1)).expert_ids.tolist() == [[1]]
    assert G.top_k_gate(np.array([[0.0, -0.0, 1.0, 1.0]]), G.GatingConfig(4, 2)).expert_ids.tolist() == [[2, 3]]
    g = G.top_k_gate(np.array([[0.4, 2.0, -1.0, 1.5]]), G.GatingConfig(4, 2))
    assert g.gate_probs[0].sum() < 1.0
    rng = np.random.default_rng(42)
    g = G.top_k_gate(rng.standard_normal((50, 8)), G.GatingConfig(8, 2))
    assert np.allclose(g.probs.sum(axis=1), 1.0, atol=1e-12)
    assert (g.expert_ids[:, 0] != g.expert_ids[:, 1]).all()


def test_gate_shape_errors():
    with pytest.raises(G.ShapeError if hasattr(G, "ShapeError") else ValueError):
        G.top_k_gate(np.zeros((4, 5)), G.GatingConfig(8, 1))
    with pytest.raises(ValueError):
        G.top_k_gate(np.zeros(5), G.GatingConfig(5, 1))


def test_plans_golden_bitwise():
    z = _load("plans.npz")
    for i in range(int(z["n"])):
        e, k, cf = z[f"p{i}_cfg"]
        cfg = G.GatingConfig(int(e), int(k), float(cf))
        lg = z[f"p{i}_logits"]
        gate = G.top_k_gate(lg, cfg)
        assert np.array_equal(gate.expert_ids, z[f"p{i}_ids"]), i
        plan = G.build_dispatch_plan(gate, cfg, lg.shape[0])
        assert plan.capacity == int(z[f"p{i}_cap"])
        assert plan.slots.dtype == np.int64
        assert np.array_equal(plan.slots, z[f"p{i}_slots"]), i
        assert np.array_equal(plan.expert_load, z[f"p{i}_load"]), i


@pytest.mark.parametrize("S,E,k,cf,skew", [
    (65536, 128, 1, 1.0, 0.0), (65536, 128, 1, 1.0, 0.5), (16384, 16, 2, 1.25, 0.5),
    (4096, 8, 1, 1.0, 0.5), (1000, 3072, 2, 0.3, 1.0), (129, 2, 2, 2.0, 0.0), (1, 4, 1, 1.0, 0.0),
])
def test_plan_random_vs_oracle(S, E, k, cf, skew):
    rng = np.random.default_rng(S + E)
    lg = (rng.standard_normal((S, E)) + rng.normal(0, skew, size=(1, E))).astype(np.float32)
    cfg = G.GatingConfig(E, k, cf)
    dev = torch.from_numpy(lg).cuda()
    gate = G.top_k_gate(dev, cfg)  # device path: fp32 comparisons
    ids_ref, gp_ref, _ = O.top_k_gate(lg.astype(np.float64), E, k)
    assert np.array_equal(gate.expert_ids.cpu().numpy(), ids_ref)
    np.testing.assert_allclose(gate.gate_probs.cpu().numpy(), gp_ref, rtol=2e-6)
    plan = G.build_dispatch_plan(gate, cfg, S)
    slots, load, cap = O.build_dispatch_plan_fast(ids_ref, E, k, cf)
    assert plan.capacity == cap
    assert np.array_equal(plan.slots.cpu().numpy(), slots)
    assert np.array_equal(plan.expert_load.cpu().numpy(), load)


def test_plan_determinism_and_empty():
    rng = np.random.default_rng(6)
    lg = rng.standard_normal((40, 4))
    cfg = G.GatingConfig(4, 2, 1.0)
    a = G.build_dispatch_plan(G.top_k_gate(lg, cfg), cfg, 40)
    b = G.build_dispatch_plan(G.top_k_gate(lg.copy(), cfg), cfg, 40)
    assert np.array_equal(a.slots, b.slots) and np.array_equal(a.gate_probs, b.gate_probs)
    cfg = G.GatingConfig(4, 1)
    plan = G.build_dispatch_plan(G.top_k_gate(np.zeros((0, 4)), cfg), cfg, 0)
    assert plan.capacity == 0 and plan.slots.shape == (0, 1)
    c = G.OpCounter()
    buf = G.scatter_tokens(np.zeros((0, 3)), plan, c)
    assert buf.data.shape == (4, 0, 3)
    assert G.combine_tokens(buf, plan, c).shape == (0, 3) and c.ops == 0


def test_scans_golden_bitwise():
    z = _load("scans.npz")
    assert G.exclusive_scan_blelloch(z["worked_in"]).tolist() == [0, 3, 4, 11, 11, 15, 16, 22]
    for i in range(int(z["n_int"])):
        got = G.exclusive_scan_blelloch(z[f"i{i}_in"])
        assert got.dtype == np.int64 and np.array_equal(got, z[f"i{i}_out"]), i
    for i in range(int(z["n_float"])):
        assert np.array_equal(G.exclusive_scan_blelloch(z[f"f{i}_in"]), z[f"f{i}_out"]), i
    with pytest.raises(ValueError):
        G.exclusive_scan_blelloch(np.zeros((2, 2)))
    assert G.exclusive_scan_blelloch(np.array([], dtype=np.int64)).shape == (0,)


def test_scan_long_vectors():
    # acceptance C5 (test_acceptance.py:168-187) plus a multi-level case
    rng = np.random.default_rng(5)
    for n in list(range(0, 300)) + [4095, 4096, 4097, 50001, 5_000_001]:
        v = rng.integers(0, 100, size=n)
        want = np.concatenate([[0], np.cumsum(v)[:-1]]) if n else np.zeros(0, np.int64)
        assert np.array_equal(G.exclusive_scan_blelloch(v), want), n


def test_scatter_combine_golden_bitwise():
    z = _load("scatter_combine.npz")
    for i in range(int(z["n"])):
        e, k, cf = z[f"s{i}_cfg"]
        e, k = int(e), int(k)
        cap = z[f"s{i}_data"].shape[1]
        s = z[f"s{i}_x"].shape[0]
        plan = G.DispatchPlan(num_tokens=s, num_experts=e, k=k, capacity=cap,
                              expert_ids=z[f"s{i}_ids"], gate_probs=z[f"s{i}_gp"],
                              slots=z[f"s{i}_slots"], expert_load=None)
        c = G.OpCounter()
        buf = G.scatter_tokens(z[f"s{i}_x"], plan, c)
        assert np.array_equal(buf.data, z[f"s{i}_data"]), i
        assert np.array_equal(buf.occupied, z[f"s{i}_occ"]), i

        class B:
            data = np.tanh(buf.data)
        comb = G.combine_tokens(B, plan, c)
        assert np.array_equal(comb, z[f"s{i}_comb"]), i
        assert c.ops == int(z[f"s{i}_ops"])


def test_scatter_combine_semantics():
    # test_gating.py:310-348
    rng = np.random.default_rng(10)
    cfg = G.GatingConfig(4, 1, 4.0)
    batch = rng.standard_normal((16, 5))
    gates = G.top_k_gate(rng.standard_normal((16, 4)), cfg)
    plan = G.build_dispatch_plan(gates, cfg, 16)
    out = G.combine_tokens(G.scatter_tokens(batch, plan), plan)
    assert np.max(np.abs(out - batch * gates.gate_probs[:, 0:1])) <= 1e-15
    cfg = G.GatingConfig(2, 1, 0.5)
    plan = G.build_dispatch_plan(G.top_k_gate(np.tile([[1.0, 0.0]], (8, 1)), cfg), cfg, 8)
    out = G.combine_tokens(G.scatter_tokens(np.ones((8, 3)), plan), plan)
    assert plan.capacity == 2 and not np.any(out[2:]) and np.all(out[:2] != 0)
    cfg = G.GatingConfig(1, 1, 1.0)
    batch = rng.standard_normal((10, 4))
    plan = G.build_dispatch_plan(G.top_k_gate(np.zeros((10, 1)), cfg), cfg, 10)
    assert np.array_equal(G.combine_tokens(G.scatter_tokens(batch, plan), plan), batch)


def test_device_tensors_stay_on_device():
    cfg = G.GatingConfig(16, 2, 1.25)
    x = torch.randn(1000, 64, device="cuda", dtype=torch.bfloat16)
    lg = torch.randn(1000, 16, device="cuda")
    gate = G.top_k_gate(lg, cfg)
    plan = G.build_dispatch_plan(gate, cfg, 1000)
    buf = G.scatter_tokens(x, plan)
    assert buf.data.is_cuda and buf.data.dtype == torch.bfloat16
    out = G.combine_tokens(buf, plan)
    # identity experts: out = x * (p0 [+ p1]) over kept choices
    kept = (plan.slots >= 0).float()
    w = (gate.gate_probs * kept).sum(1, keepdim=True)
    torch.testing.assert_close(out.float(), x.float() * w, rtol=1e-2, atol=1e-2)


def test_ep_plan_kernel_matches_host_plan():
    """moe_ep_plan (device exchange plan of the peer-memory EP transport) against a
    NumPy restatement, for simulated worlds of 2/4/8 ranks (pure function of the
    all-gathered counts, so one GPU covers every rank's view)."""
    from paper_2201_05596_b200 import _lib

    rng = np.random.default_rng(11)
    for world in (1, 2, 4, 8):
        E = 16 * world
        counts = rng.integers(0, 700, size=(world, E)).astype(np.int32)
        cap = int(counts.sum(0).mean())
        e_loc = E // world
        base = np.zeros_like(counts, dtype=np.int64)
        base[1:] = np.cumsum(counts, 0)[:-1]
        kept = np.clip(cap - base, 0, counts)
        for rank in range(world):
            c_d = torch.from_numpy(counts).cuda().reshape(-1)
            out = [torch.empty(E, dtype=torch.int32, device="cuda") for _ in range(2)]
            seg = [torch.empty(e_loc, dtype=torch.int32, device="cuda") for _ in range(2)]
            rr = torch.empty(1, dtype=torch.int32, device="cuda")
            _lib.call("moe_ep_plan", c_d.data_ptr(), world, rank, E, cap, out[0].data_ptr(),
                      out[1].data_ptr(), seg[0].data_ptr(), seg[1].data_ptr(), rr.data_ptr(),
                      _lib.stream_ptr())
            assert np.array_equal(out[0].cpu().numpy(), base[rank])
            # expert-major receive layout on each owner: [local expert][source][slot]
            row_base = np.zeros(E, dtype=np.int64)
            for e in range(E):
                o, el = divmod(e, e_loc)
                blk = kept[:, o * e_loc:o * e_loc + el].sum()
                row_base[e] = blk + kept[:rank, e].sum()
            assert np.array_equal(out[1].cpu().numpy(), row_base)
            mine = kept[:, rank * e_loc:(rank + 1) * e_loc].sum(0)
            assert np.array_equal(seg[1].cpu().numpy(), mine)
            assert np.array_equal(seg[0].cpu().numpy(), np.concatenate([[0], np.cumsum(mine)[:-1]]))
            assert int(rr.item()) == int(mine.sum())


def test_load_balance_loss_golden_and_api():
    """arch.load_balance_loss on the device against the reference's values
    (tests/golden/plans.npz, generated with moekit.arch.load_balance_loss)."""
    from paper_2201_05596_b200 import arch as A

    z = _load("plans.npz")
    for i in range(int(z["n"])):
        e, k, cf = z[f"p{i}_cfg"]
        cfg = G.GatingConfig(int(e), int(k), float(cf))
        lg = z[f"p{i}_logits"]
        gate = G.top_k_gate(lg, cfg)
        plan = G.build_dispatch_plan(gate, cfg, lg.shape[0])
        got = A.load_balance_loss(plan, gate.probs)
        assert abs(got - float(z[f"p{i}_lbl"])) <= 1e-12 * max(1.0, abs(got)), i
    with pytest.raises(ValueError):
        A.load_balance_loss(plan, np.zeros((3, 3)))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_fused_aux_loss_matches_oracle(dtype):
    """The gate epilogue's softmax column sums + the scan's pre-drop counts give
    the same load-balance loss as the oracle on the layer's own logits."""
    from paper_2201_05596_b200 import arch as A

    S, M, E, k = 3000, 256, 16, 2
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, gating=G.GatingConfig(E, k, 1.0))
    p = A.init_layer_params(spec, np.random.default_rng(4))
    p.gate_w.value[:] += np.random.default_rng(5).normal(0, 0.3, (1, E))
    layer = A.MoeLayer(spec, p, dtype=dtype)
    layer.aux_loss = True
    x = torch.randn(S, M, device="cuda").to(dtype)
    logits = torch.empty(S, E, device="cuda")
    layer(x, logits_out=logits)
    got = float(layer.last_aux_loss.item())
    ids, _, probs = O.top_k_gate(logits.double().cpu().numpy(), E, k)
    want = O.load_balance_loss(ids, probs, E, k)
    assert abs(got - want) <= 1e-5 * want


def _nan_inf_rows(E, rng):
    """Logit rows numpy's stable argsort orders specially: NaN last, -inf before
    NaN, +-0 ties, a single finite value among -inf, all NaN, all -inf."""
    ninf, nan = -np.inf, np.nan
    rows = [np.full(E, nan), np.full(E, ninf), np.where(np.arange(E) % 2, ninf, nan)]
    r = np.full(E, ninf)
    r[E - 1] = 0.5
    rows.append(r)
    r = np.full(E, nan)
    r[E // 2] = ninf
    rows.append(r)
    r = rng.standard_normal(E)
    r[::3] = nan
    rows.append(r)
    r = rng.standard_normal(E)
    r[1] = np.inf
    rows.append(r)
    r = np.zeros(E)
    r[::2] = -0.0
    rows.append(r)
    return np.stack(rows)


@pytest.mark.parametrize("E,k", [(4, 1), (4, 2), (8, 2), (128, 2), (300, 1)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_gate_nan_inf_rows_match_stable_argsort(E, k, dt):
    """a NaN / -inf row must route like np.argsort(-logits,
    kind="stable") (gating.py:159-161), never to an index outside [0, E)."""
    rng = np.random.default_rng(E + k)
    lg = np.concatenate([_nan_inf_rows(E, rng), rng.standard_normal((40, E))]).astype(dt)
    cfg = G.GatingConfig(E, k)
    with np.errstate(invalid="ignore"):
        want = np.argsort(-lg.astype(np.float64), axis=1, kind="stable")[:, :k]
    for inp in (lg, torch.from_numpy(lg).cuda()):
        g = G.top_k_gate(inp, cfg)
        ids = g.expert_ids.cpu().numpy() if torch.is_tensor(g.expert_ids) else g.expert_ids
        assert np.array_equal(ids, want)
        plan = G.build_dispatch_plan(g, cfg, lg.shape[0])
        s_ref, l_ref, _ = O.build_dispatch_plan(want, E, k, 1.0)
        slots = plan.slots.cpu().numpy() if torch.is_tensor(plan.slots) else plan.slots
        assert np.array_equal(slots, s_ref)


@pytest.mark.parametrize("E,k", [(8, 1), (8, 2), (128, 1), (128, 2), (33, 2)])
def test_fused_gate_nan_rows(E, k):
    """The tcgen05 gate epilogue: tokens whose logits are NaN / +-inf (NaN or
    inf activations) route like the stable argsort of the logits it emitted."""
    from paper_2201_05596_b200 import arch as A

    S, M = 700, 64
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, gating=G.GatingConfig(E, k, 1.0))
    p = A.init_layer_params(spec, np.random.default_rng(E))
    layer = A.MoeLayer(spec, p, dtype=torch.bfloat16)
    x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
    x[3] = float("nan")
    x[130, 5] = float("nan")
    x[131, 0] = float("inf")
    x[260] = float("-inf")
    x[261, :8] = float("inf")
    logits = torch.empty(S, E, device="cuda")
    layer(x, logits_out=logits)
    torch.cuda.synchronize()
    lg = logits.double().cpu().numpy()
    assert np.isnan(lg[3]).all()
    with np.errstate(invalid="ignore"):
        want = np.argsort(-lg, axis=1, kind="stable")[:, :k]
    ids, gp, slots, load, cap = layer.plan(S)
    assert np.array_equal(ids.cpu().numpy(), want)
    s_ref, l_ref, c_ref = O.build_dispatch_plan(want, E, k, 1.0)
    assert np.array_equal(slots.cpu().numpy(), s_ref)
    assert np.array_equal(load.cpu().numpy(), l_ref)


def test_plan_hand_built_ids():
    """a hand-built gate may hold ids outside [0, E) (they match no
    expert's indicator and stay DROPPED, gating.py:229-230) or repeat an
    expert within a token's k=2 choices (token-major: slots s and s+1)."""
    rng = np.random.default_rng(5)
    for k in (1, 2):
        E, S = 6, 300
        ids = rng.integers(-2, E + 2, size=(S, k)).astype(np.int64)
        ids[::7, :] = 3  # repeated choice (k=2) / hot expert
        ids[5, 0] = 2 ** 33 + 1  # would alias to 1 if narrowed to int32
        gate = G.TopKGate(expert_ids=ids, gate_probs=np.full((S, k), 0.5),
                          probs=np.full((S, E), 1.0 / E))
        cfg = G.GatingConfig(E, k, 1.5)
        s_ref, l_ref, c_ref = O.build_dispatch_plan(ids, E, k, 1.5)
        for g in (gate, G.TopKGate(torch.from_numpy(ids).cuda(), torch.full((S, k), 0.5).cuda(),
                                   torch.full((S, E), 1.0 / E).cuda())):
            plan = G.build_dispatch_plan(g, cfg, S)
            slots = plan.slots.cpu().numpy() if torch.is_tensor(plan.slots) else plan.slots
            load = (plan.expert_load.cpu().numpy() if torch.is_tensor(plan.expert_load)
                    else plan.expert_load)
            assert plan.capacity == c_ref
            assert np.array_equal(slots, s_ref), k
            assert np.array_equal(load, l_ref), k
