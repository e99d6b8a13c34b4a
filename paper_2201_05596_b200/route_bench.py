"""GPU-backed ``route-bench`` verb.

Mirrors ``moekit route-bench`` (cli.py:246-306): the same JSON options
(tokens, experts, k, capacity_factor, instances), the same per-instance RNG
draws (default_rng(seed + i): logits (tokens, experts), x (tokens, 32)), and
the same CSV columns, plus ``gpu_us``: the device time of the table-driven
routing pipeline (top_k_gate -> build_dispatch_plan -> scatter_tokens ->
combine_tokens, float64 on the B200) measured with CUDA events — the wall
time the reference's "throughput microbenchmark" never reported
(README.md:70). ``max_abs_err`` compares the table path with the literal
one-hot einsum contraction (gating.py:315-377), evaluated here with torch on
the device; ``op_ratio`` uses the reference's OpCounter convention.

    python -m paper_2201_05596_b200.route_bench [--config c.json] [--seed N] [--out f.csv]

Exit codes follow cli.py:53-56 (0 ok, 2 config error).
"""

from __future__ import annotations

import argparse
import csv
import json
import sys

import numpy as np
import torch

from . import gating
from .arch import load_balance_loss

EXIT_OK, EXIT_CONFIG = 0, 2
DEFAULT_SEED = 42
HEADER = ["instance", "tokens", "experts", "k", "capacity", "kept", "dropped", "balance_loss",
          "max_abs_err", "op_ratio", "gpu_us"]
OPTIONS = {"tokens", "experts", "k", "capacity_factor", "instances"}


class ConfigError(ValueError):
    pass


def _fmt(x) -> str:
    return f"{x:.10g}" if isinstance(x, float) else str(x)


def _onehot_mask(ids: torch.Tensor, E: int, cap: int) -> torch.Tensor:
    """(S, E, c) one-hot dispatch mask from an independent cumsum (gating.py:315-331)."""
    S, k = ids.shape
    flat = ids.reshape(-1).long()
    hot = torch.nn.functional.one_hot(flat, E).to(torch.float64)
    running = torch.cumsum(hot, 0) - hot
    mask = torch.zeros((S * k, E, cap), dtype=torch.float64, device=ids.device)
    r, c = torch.nonzero(hot, as_tuple=True)
    sl = running[r, c].long()
    ok = sl < cap
    mask[r[ok], c[ok], sl[ok]] = 1.0
    return mask.reshape(S, k, E, cap).sum(1)


def run(opts: dict, seed: int) -> list[list]:
    tokens = opts.get("tokens", 256)
    experts = opts.get("experts", 8)
    k = opts.get("k", 1)
    cf = opts.get("capacity_factor", 1.0)
    instances = opts.get("instances", 20)
    try:
        cfg = gating.GatingConfig(num_experts=experts, k=k, capacity_factor=cf)
    except ValueError as e:
        raise ConfigError(f"bad routing options: {e}") from e
    hidden = 32
    dev = torch.device("cuda", torch.cuda.current_device())
    rows = []
    for i in range(instances):
        rng = np.random.default_rng(seed + i)
        logits = torch.from_numpy(rng.standard_normal((tokens, experts))).to(dev)
        x = torch.from_numpy(rng.standard_normal((tokens, hidden))).to(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        mapped = gating.OpCounter()
        e0.record()
        gate = gating.top_k_gate(logits, cfg)
        plan = gating.build_dispatch_plan(gate, cfg, tokens)
        bufs = gating.scatter_tokens(x, plan, counter=mapped)
        combined = gating.combine_tokens(bufs, plan, counter=mapped)
        e1.record()
        torch.cuda.synchronize()
        gpu_us = e0.elapsed_time(e1) * 1e3
        # one-hot contraction reference path (S*E*c*M work per transform)
        cap = plan.capacity
        oracle_ops = tokens * experts * cap * hidden * 2
        if tokens and cap:
            mask = _onehot_mask(gate.expert_ids, experts, cap)
            obuf = torch.einsum("sec,sm->ecm", mask, x)
            kept = plan.slots >= 0
            w = torch.zeros((tokens, experts), dtype=torch.float64, device=dev)
            for j in range(k):
                w[torch.arange(tokens, device=dev), gate.expert_ids[:, j].long()] += torch.where(
                    kept[:, j], gate.gate_probs[:, j], torch.zeros_like(gate.gate_probs[:, j]))
            oout = torch.einsum("sec,ecm->sm", mask * w[:, :, None], obuf)
            err = float((combined - oout).abs().max().item())
        else:
            err = 0.0
        n_kept = int((plan.slots >= 0).sum().item())
        rows.append([i, tokens, experts, k, cap, n_kept, tokens * k - n_kept,
                     _fmt(load_balance_loss(plan, gate.probs)), _fmt(err),
                     _fmt(oracle_ops / mapped.ops if mapped.ops else 0.0), _fmt(gpu_us)])
    return rows


def main(argv: list[str] | None = None) -> int:
    ap = argparse.ArgumentParser(prog="route_bench")
    ap.add_argument("--config")
    ap.add_argument("--out")
    ap.add_argument("--seed", type=int, default=None)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    try:
        config = {}
        if args.config:
            try:
                config = json.load(open(args.config))
            except (OSError, json.JSONDecodeError) as e:
                raise ConfigError(f"cannot read config {args.config}: {e}") from e
            if not isinstance(config, dict):
                raise ConfigError("config root must be a JSON object")
            unknown = set(config) - {"seed", "model", "cluster", "options"}
            if unknown:
                raise ConfigError(f"unknown config keys: {sorted(unknown)}")
        opts = config.get("options") or {}
        if not isinstance(opts, dict):
            raise ConfigError("options must be a JSON object")
        unknown = set(opts) - OPTIONS
        if unknown:
            raise ConfigError(f"unknown route-bench options keys: {sorted(unknown)}")
        seed = args.seed if args.seed is not None else config.get("seed", DEFAULT_SEED)
        if not isinstance(seed, int):
            raise ConfigError("seed must be an integer")
        rows = run(opts, seed)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    out = open(args.out, "w", newline="") if args.out else sys.stdout
    w = csv.writer(out)
    w.writerow(HEADER)
    w.writerows(rows)
    if args.out:
        out.close()
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
