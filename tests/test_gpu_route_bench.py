"""GPU route-bench verb against the reference CLI's own route-bench output
(tests/golden/route_bench_*.csv, generated with moekit.cli.main) and the
checks of the reference's tests/test_cli.py:122-149."""

import csv
import json
import os

import pytest

from paper_2201_05596_b200 import route_bench
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASES = [("route_bench_a.csv", {"tokens": 300, "experts": 8, "k": 2, "capacity_factor": 1.0,
                                "instances": 5}, 7),
         ("route_bench_b.csv", {"tokens": 1000, "experts": 16, "k": 1, "capacity_factor": 0.5,
                                "instances": 3}, 11)]


def _run(tmp_path, opts, seed):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"seed": seed, "options": opts}))
    out = tmp_path / "o.csv"
    assert route_bench.main(["--config", str(cfg), "--out", str(out)]) == 0
    return list(csv.DictReader(open(out)))


@pytest.mark.parametrize("name,opts,seed", CASES)
def test_matches_reference_cli(tmp_path, name, opts, seed):
    ref = list(csv.DictReader(open(os.path.join(GOLDEN, name))))
    got = _run(tmp_path, opts, seed)
    assert len(got) == len(ref)
    for g, r in zip(got, ref):
        for key in ("instance", "tokens", "experts", "k", "capacity", "kept", "dropped"):
            assert g[key] == r[key], key
        assert abs(float(g["balance_loss"]) - float(r["balance_loss"])) <= 1e-9
        assert float(g["max_abs_err"]) <= 1e-9
        assert abs(float(g["op_ratio"]) - float(r["op_ratio"])) <= 1e-9
        assert float(g["gpu_us"]) > 0
        assert int(g["kept"]) + int(g["dropped"]) == opts["tokens"] * opts["k"]


def test_determinism_and_config_errors(tmp_path):
    a = _run(tmp_path, CASES[0][1], 3)
    b = _run(tmp_path, CASES[0][1], 3)
    strip = lambda rows: [{k: v for k, v in r.items() if k != "gpu_us"} for r in rows]  # noqa: E731
    assert strip(a) == strip(b)
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"options": {"tokens": 10, "bogus": 1}}))
    assert route_bench.main(["--config", str(bad)]) == 2
    bad.write_text(json.dumps({"options": {"k": 3}}))
    assert route_bench.main(["--config", str(bad)]) == 2
