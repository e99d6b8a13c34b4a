"""The reference's acceptance criteria for this path (pkg/tests/test_acceptance.py
C4 and C5), run against the B200 implementation through its public API with
the same generators, seeds and limits:

  C4  1000 random routing instances (seed 2024): scatter / combine through the
      mapping table equal the one-hot einsum oracles within 1e-9, the oracle's
      op count is E x the table's (+-20%), all in < 60 s;
  C5  the exclusive scan on every length 0..1025 and 100 long vectors (seed 5)
      equals the sequential scan, in < 5 s.
"""

import time

import numpy as np
import pytest

from oracle import moe_oracle as O
from paper_2201_05596_b200 import gating

pytestmark = pytest.mark.gpu


def test_c04_routing_oracle_equivalence():
    start = time.monotonic()
    rng = np.random.default_rng(2024)
    hidden = 8
    worst_err, ratio_ok = 0.0, True
    for _ in range(1000):
        s = int(rng.integers(1, 257))
        e = int(rng.integers(1, 17))
        k = int(rng.integers(1, 3)) if e >= 2 else 1
        cf = float(rng.choice([0.5, 1.0, 2.0]))
        cfg = gating.GatingConfig(num_experts=e, k=k, capacity_factor=cf)
        gate = gating.top_k_gate(rng.standard_normal((s, e)), cfg)
        plan = gating.build_dispatch_plan(gate, cfg, s)
        x = rng.standard_normal((s, hidden))
        mapped = gating.OpCounter()
        buffers = gating.scatter_tokens(x, plan, counter=mapped)
        combined = gating.combine_tokens(buffers, plan, counter=mapped)
        cap = cfg.capacity(s)
        obuf = O.sparse_dispatch_oracle(x, gate.expert_ids, e, cap)
        oout = O.sparse_combine_oracle(obuf, gate.expert_ids, gate.gate_probs, e, cap)
        oracle_ops = 2 * s * e * cap * hidden  # S*E*c*M per one-hot contraction (gating.py:345, :376)
        worst_err = max(worst_err, float(np.max(np.abs(buffers.data - obuf))),
                        float(np.max(np.abs(combined - oout))))
        if mapped.ops:
            ratio = oracle_ops / mapped.ops
            ratio_ok &= 0.8 * e <= ratio <= 1.2 * e
    elapsed = time.monotonic() - start
    assert worst_err <= 1e-9, worst_err
    assert ratio_ok
    assert elapsed < 60.0, elapsed


def _sequential(v):
    out = np.zeros_like(v)
    run = 0
    for i, x in enumerate(v):
        out[i] = run
        run += x
    return out


def test_c05_scan_correctness():
    rng = np.random.default_rng(5)
    cases = [rng.integers(0, 7, size=n) for n in range(1026)]
    cases += [rng.integers(0, 100, size=int(rng.integers(2000, 50001))) for _ in range(100)]
    gating.exclusive_scan_blelloch(cases[5])  # warm the library outside the timed loop
    start = time.monotonic()
    got = [gating.exclusive_scan_blelloch(v) for v in cases]
    elapsed = time.monotonic() - start
    bad = sum(not np.array_equal(g, np.concatenate([[0], np.cumsum(v)[:-1]]) if len(v) else v)
              for g, v in zip(got, cases))
    assert bad == 0
    assert all(np.array_equal(got[n], _sequential(cases[n])) for n in (0, 1, 2, 17, 1025))
    assert elapsed < 5.0, elapsed
