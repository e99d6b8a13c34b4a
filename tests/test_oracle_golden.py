"""Pin the CPU oracle (oracle/moe_oracle.py) to golden vectors produced by the
reference itself (tests/golden/make_golden.py). CPU only."""

import os

import numpy as np

from oracle import moe_oracle as O
from tests.conftest import GOLDEN


def _load(name):
    return np.load(os.path.join(GOLDEN, name))


def test_gate_kats_bitwise():
    z = _load("gate_kats.npz")
    for i in range(int(z["n"])):
        lg, k = z[f"c{i}_logits"], int(z[f"c{i}_k"])
        ids, gp, probs = O.top_k_gate(lg, lg.shape[1], k)
        assert np.array_equal(ids, z[f"c{i}_ids"]), i
        assert np.array_equal(gp, z[f"c{i}_gp"]), i
        assert np.array_equal(probs, z[f"c{i}_probs"]), i


def test_gate_kat_values():
    # test_gating.py:65-83 literal expectations
    assert O.top_k_gate(np.array([[1.0, 3.0, 2.0]]), 3, 1)[0].tolist() == [[1]]
    assert O.top_k_gate(np.array([[1.0, 3.0, 2.0]]), 3, 2)[0].tolist() == [[1, 2]]
    assert O.top_k_gate(np.array([[5.0, 5.0, 1.0]]), 3, 2)[0].tolist() == [[0, 1]]
    assert O.top_k_gate(np.array([[2.0, 7.0, 7.0, 7.0]]), 4, 1)[0].tolist() == [[1]]


def test_scans_bitwise():
    z = _load("scans.npz")
    assert O.exclusive_scan_blelloch(z["worked_in"]).tolist() == [0, 3, 4, 11, 11, 15, 16, 22]
    for i in range(int(z["n_int"])):
        got = O.exclusive_scan_blelloch(z[f"i{i}_in"])
        assert got.dtype == np.int64
        assert np.array_equal(got, z[f"i{i}_out"]), i
    for i in range(int(z["n_float"])):
        got = O.exclusive_scan_blelloch(z[f"f{i}_in"])
        assert np.array_equal(got, z[f"f{i}_out"]), i  # same tree order -> bitwise


def test_plans_bitwise():
    z = _load("plans.npz")
    for i in range(int(z["n"])):
        e, k, cf = z[f"p{i}_cfg"]
        e, k = int(e), int(k)
        ids, gp, probs = O.top_k_gate(z[f"p{i}_logits"], e, k)
        assert np.array_equal(ids, z[f"p{i}_ids"])
        assert np.array_equal(gp, z[f"p{i}_gp"])
        slots, load, cap = O.build_dispatch_plan(ids, e, k, float(cf))
        assert cap == int(z[f"p{i}_cap"])
        assert np.array_equal(slots, z[f"p{i}_slots"]), i
        assert np.array_equal(load, z[f"p{i}_load"]), i
        s2, l2, c2 = O.build_dispatch_plan_fast(ids, e, k, float(cf))
        assert np.array_equal(s2, slots) and np.array_equal(l2, load) and c2 == cap
        assert O.load_balance_loss(ids, probs, e, k) == float(z[f"p{i}_lbl"])
    for e, k, cf, s, cap in z["capacity_table"]:
        assert O.capacity(int(e), int(k), float(cf), int(s)) == int(cap)


def test_scatter_combine():
    z = _load("scatter_combine.npz")
    for i in range(int(z["n"])):
        e, k, cf = z[f"s{i}_cfg"]
        e = int(e)
        cap = z[f"s{i}_data"].shape[1]
        data, occ = O.scatter_tokens(z[f"s{i}_x"], z[f"s{i}_ids"], z[f"s{i}_slots"], e, cap)
        assert np.array_equal(data, z[f"s{i}_data"])
        assert np.array_equal(occ, z[f"s{i}_occ"])
        comb = O.combine_tokens(np.tanh(data), z[f"s{i}_ids"], z[f"s{i}_slots"], z[f"s{i}_gp"])
        assert np.array_equal(comb, z[f"s{i}_comb"])
        # one-hot oracles agree with the table path (test_gating.py:292-308): dispatch
        # bitwise, combine within 1e-12
        assert np.array_equal(O.sparse_dispatch_oracle(z[f"s{i}_x"], z[f"s{i}_ids"], e, cap), data)
        oc = O.sparse_combine_oracle(np.tanh(data), z[f"s{i}_ids"], z[f"s{i}_gp"], e, cap)
        assert np.max(np.abs(oc - z[f"s{i}_comb"]), initial=0.0) <= 1e-12


def _layer_case(z, i):
    s, m, e, k, cf, res = z[f"l{i}_cfg"]
    e, k = int(e), int(k)
    experts = [(z[f"l{i}_w1"][j], z[f"l{i}_b1"][j], z[f"l{i}_w2"][j], z[f"l{i}_b2"][j])
               for j in range(e)]
    shared = None
    if res:
        shared = (z[f"l{i}_sw1"], z[f"l{i}_sb1"], z[f"l{i}_sw2"], z[f"l{i}_sb2"])
    return z[f"l{i}_x"], z[f"l{i}_gate_w"], experts, shared, e, k, float(cf)


def test_layers_match_reference():
    z = _load("layers.npz")
    for i in range(int(z["n"])):
        x, gw, experts, shared, e, k, cf = _layer_case(z, i)
        out = O.forward_layer(x, gw, experts, shared, e, k, cf)
        assert np.max(np.abs(out - z[f"l{i}_out"])) <= 1e-12, i


def test_layer_sampled_matches_full():
    z = _load("layers.npz")
    for i in range(int(z["n"])):
        x, gw, experts, shared, e, k, cf = _layer_case(z, i)
        logits = x @ gw
        full = O.forward_layer_with_logits(x, logits, experts, shared, e, k, cf)
        subset = list(range(0, e, 2)) or [0]
        tok, rows = O.forward_layer_sampled(x, logits, experts, shared, e, k, cf, subset)
        assert np.max(np.abs(rows - full[tok]), initial=0.0) <= 1e-12


def test_dropped_tokens_ride_skip():
    # test_arch.py:267-275
    z = _load("layers.npz")
    x, gw, experts, shared, e, k, cf = _layer_case(z, 4)
    out = O.forward_layer(x, gw, experts, shared, e, k, cf)
    assert np.all(out == x, axis=1).sum() >= 4


def test_backward_oracle_matches_reference_tape():
    """The oracle's closed-form backward against moekit's GradTape (golden)."""
    z = _load("layer_grads.npz")
    for i in range(int(z["n"])):
        s, m, e, k, cf, res = z[f"g{i}_cfg"]
        e, k = int(e), int(k)
        f64 = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
        experts = [(f64(z[f"g{i}_w1"][j]), f64(z[f"g{i}_b1"][j]), f64(z[f"g{i}_w2"][j]),
                    f64(z[f"g{i}_b2"][j])) for j in range(e)]
        shared = None
        if res:
            shared = tuple(f64(z[f"g{i}_s{n}"]) for n in ("w1", "b1", "w2", "b2"))
        x, gw = f64(z[f"g{i}_x"]), f64(z[f"g{i}_gate_w"])
        g = O.forward_layer_backward(x, x @ gw, gw, experts, shared, e, k, float(cf),
                                     f64(z[f"g{i}_G"]))
        tol = lambda want: 1e-6 * (np.abs(want) + np.abs(want).max())  # float32-stored fixtures  # noqa: E731
        for key, want in (("x", z[f"g{i}_dx"]), ("gate_w", z[f"g{i}_dgate_w"])):
            assert np.all(np.abs(g[key] - want) <= tol(want)), (i, key)
        for n in ("w1", "b1", "w2", "b2"):
            want = z[f"g{i}_d{n}"]
            got = np.stack(g[n]).reshape(want.shape)
            assert np.all(np.abs(got - want) <= tol(want)), (i, n)
        if res:
            for n in ("w1", "b1", "w2", "b2"):
                want = z[f"g{i}_ds{n}"]
                assert np.all(np.abs(g["shared"][n].reshape(want.shape) - want) <= tol(want))
