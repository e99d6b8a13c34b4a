"""Multi-GPU expert-parallel parity (run under torchrun, one rank per GPU).

Every rank builds the same full parameters; rank r runs the expert-parallel
layer on its token shard and compares with the single-GPU layer run on the
whole batch. Routing (ids, global slots) and outputs must be bit-identical:
both paths evaluate each row with the same kernels in the same order.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2201_05596_b200 import arch as A  # noqa: E402
from paper_2201_05596_b200.ep import EPMoeLayer, SlicedEPMoeLayer  # noqa: E402
from paper_2201_05596_b200.gating import GatingConfig  # noqa: E402

SAME_DEVICE = os.environ.get("EP_SAME_DEVICE") == "1"


def make_params(M, E, residual, skew, g, dev):
    F = 4 * M
    gw = torch.randn(M, E, device=dev, generator=g) * 0.1
    gw += torch.randn(1, E, device=dev, generator=g) * skew
    ex = [A.FfnParams(torch.randn(M, F, device=dev, generator=g) * 0.1,
                      torch.randn(1, F, device=dev, generator=g) * 0.05,
                      torch.randn(F, M, device=dev, generator=g) * 0.1,
                      torch.randn(1, M, device=dev, generator=g) * 0.05) for _ in range(E)]
    sh = None
    if residual:
        sh = A.FfnParams(torch.randn(M, F, device=dev, generator=g) * 0.1,
                         torch.zeros(1, F, device=dev), torch.randn(F, M, device=dev, generator=g) * 0.1,
                         torch.zeros(1, M, device=dev))
    return A.MoeLayerParams(gate_w=gw, experts=tuple(ex), shared=sh)


def run_sliced(S_grp, M, E, k, cf, skew, seed, L):
    """Tensor-sliced groups + expert slicing vs the single-GPU layer on the
    concatenated group shards: routing bit-exact, outputs to bf16 tolerance
    (the slices' partial sums are rounded to bf16 before the all-reduce)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    Q = world // L
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=False,
                       gating=GatingConfig(E, k, cf))
    g = torch.Generator(device=dev).manual_seed(seed)
    params = make_params(M, E, False, skew, g, dev)
    x_all = torch.randn(S_grp * Q, M, device=dev, generator=g).to(torch.bfloat16)
    full = A.MoeLayer(spec, params, dtype=torch.bfloat16, device=dev, fuse_combine=False)
    want = full(x_all)
    ids_f, gp_f, slots_f, load_f, cap_f = full.plan(S_grp * Q)
    layer = SlicedEPMoeLayer.from_params(spec, params, tensor_slice=L)
    q = rank // L
    lo, hi = q * S_grp, (q + 1) * S_grp
    got = layer(x_all[lo:hi].clone())
    got = layer(x_all[lo:hi].clone())
    torch.cuda.synchronize()
    ids_e, gp_e, slots_e, plan = layer.plan(S_grp)
    assert plan.cap == cap_f
    assert torch.equal(ids_e, ids_f[lo:hi]), "ids differ"
    assert torch.equal(slots_e, slots_f[lo:hi]), "global slots differ"
    e_loc = E // Q
    assert np.array_equal(plan.expert_load, load_f[q * e_loc:(q + 1) * e_loc].cpu().numpy())
    w = want[lo:hi].double()
    rms = w.pow(2).mean().sqrt()
    excess = ((got.double() - w).abs() - 2e-2 * (w.abs() + rms)).max().item()
    assert excess <= 0, f"sliced output off by {excess}"
    # every member of a group holds the same output
    peers = [torch.empty_like(got) for _ in range(world)]
    if SAME_DEVICE:  # gloo: host tensors
        hp = [torch.empty_like(got, device="cpu") for _ in range(world)]
        dist.all_gather(hp, got.cpu())
        peers = [h.to(got.device) for h in hp]
    else:
        dist.all_gather(peers, got)
    for u in range(L):
        assert torch.equal(peers[q * L + u], got), "group members disagree"
    st = layer.exchanger.last_stats
    return st


def run_case(S_loc, M, E, k, cf, residual, skew, seed, transport="auto", schedule="flat",
             gpus_per_node=None, chunks=1):
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=residual,
                       gating=GatingConfig(E, k, cf))
    g = torch.Generator(device=dev).manual_seed(seed)
    params = make_params(M, E, residual, skew, g, dev)
    x_all = torch.randn(S_loc * world, M, device=dev, generator=g).to(torch.bfloat16)
    # the p2p transport fuses combine into GEMM2 like the single-GPU k=1 path;
    # the nccl transport uses the separate combine kernel
    full = A.MoeLayer(spec, params, dtype=torch.bfloat16, device=dev,
                      fuse_combine=(transport == "p2p"))
    want = full(x_all)
    ids_f, gp_f, slots_f, load_f, cap_f = full.plan(S_loc * world)
    ep = EPMoeLayer.from_params(spec, params, transport=transport, schedule=schedule,
                                gpus_per_node=gpus_per_node, chunks=chunks)
    lo, hi = rank * S_loc, (rank + 1) * S_loc
    got = ep(x_all[lo:hi].clone())
    got = ep(x_all[lo:hi].clone())  # second call: buffer reuse / slot alternation
    torch.cuda.synchronize()
    if hasattr(ep, "check_errors"):
        ep.check_errors()
    ids_e, gp_e, slots_e, plan = ep.plan(S_loc)
    assert plan.cap == cap_f, (plan.cap, cap_f)
    assert torch.equal(ids_e, ids_f[lo:hi]), "ids differ"
    assert torch.equal(slots_e, slots_f[lo:hi]), "global slots differ"
    e0 = rank * (E // world)
    assert np.array_equal(plan.expert_load, load_f[e0:e0 + E // world].cpu().numpy())
    if not torch.equal(got, want[lo:hi]):
        err = (got.float() - want[lo:hi].float()).abs().max().item()
        raise AssertionError(f"EP output differs from single-GPU output (max abs {err})")
    if transport == "p2p":  # the whole EP forward (NCCL all-gather + peer barriers) as a graph
        g = ep.graphed(S_loc)
        for _ in range(2):
            if not torch.equal(g(x_all[lo:hi]), want[lo:hi]):
                raise AssertionError("graph replay of the EP layer differs")
        torch.cuda.synchronize()
        ep.check_errors()
    dropped = int((slots_e < 0).sum())
    return dropped


def main():
    if SAME_DEVICE:
        # every rank on cuda:0 (the driver's 1-GPU test box): gloo bootstraps the
        # ranks (NCCL refuses two ranks on one device), the p2p transport maps
        # the other processes' regions with same-device cudaIpc, and its counts
        # all-gather and barriers run over that peer memory exactly as on NVLink
        dist.init_process_group("gloo")
        torch.cuda.set_device(0)
    else:
        dist.init_process_group("nccl")
        torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    world = dist.get_world_size()
    cases = [
        (4096, 1024, 16, 2, 1.25, False, 0.5, 1),
        (3000, 512, 8 * world, 1, 1.0, True, 1.0, 2),
        (2048, 2048, 32, 1, 1.0, False, 0.0, 3),
        (700, 256, 4 * world, 2, 0.6, False, 2.0, 4),
        (2500, 1024, 16, 1, 0.8, False, 1.0, 5),
    ]
    for c in cases:
        for transport in ("nccl", "p2p"):
            dropped = run_case(*c, transport=transport)
            if dist.get_rank() == 0:
                print(f"ep ok same_device={int(SAME_DEVICE)} world={world} transport={transport} case={c} "
                      f"dropped_on_rank0={dropped}", flush=True)
    # seeded random configurations, both transports where they apply
    rng = np.random.default_rng(2024 + world)
    for i in range(4):
        S_loc = int(rng.integers(1, 40)) * 64 + int(rng.integers(0, 64))
        M = int(rng.choice([256, 512, 1024]))
        E = world * int(rng.integers(1, 9))
        k = 1 if E == 1 else int(rng.choice([1, 2]))
        cf = float(rng.uniform(0.5, 1.5))
        residual = bool(rng.random() < 0.3)
        c = (S_loc, M, E, k, cf, residual, float(rng.uniform(0, 1.5)), 100 + i)
        for transport in ("nccl", "p2p"):
            run_case(*c, transport=transport)
            if dist.get_rank() == 0:
                print(f"ep ok same_device={int(SAME_DEVICE)} world={world} random-case via {transport} case={c}", flush=True)
    # chunked p2p (dispatch / pull of neighbouring chunks beside the GEMMs): bit-identical
    for c in [(2048, 2048, 32, 1, 1.0, False, 0.0, 3), (2560, 1024, 16, 1, 0.8, False, 1.0, 5)]:
        for chunks in (2, 4):
            if c[0] % (chunks * 128):
                continue
            dropped = run_case(*c, transport="p2p", chunks=chunks)
            if dist.get_rank() == 0:
                print(f"ep ok same_device={int(SAME_DEVICE)} world={world} transport=p2p-chunked chunks={chunks} case={c} "
                      f"dropped_on_rank0={dropped}", flush=True)
    # hierarchical node/rail schedule (2 "nodes" of world/2 GPUs): bit-identical too
    if world % 2 == 0:
        for c in cases[:2] + cases[3:4]:
            run_case(*c, transport="nccl", schedule="hierarchical", gpus_per_node=world // 2)
            if dist.get_rank() == 0:
                print(f"ep ok same_device={int(SAME_DEVICE)} world={world} schedule=hierarchical G={world // 2} case={c}",
                      flush=True)
    # tensor-sliced groups with expert slicing (coordinated exchange)
    sl_cases = [(2048, 1024, 8, 1, 1.0, 0.5, 11, 2), (1500, 512, 4, 2, 0.8, 1.0, 12, 2),
                (1024, 1024, max(world // 2, 1), 1, 1.25, 0.0, 13, 2),  # p > E: one expert per group
                (1000, 512, 8, 2, 1.0, 0.5, 14, world)]
    for c in sl_cases:
        if world % c[-1] or c[2] % (world // c[-1]):
            continue
        st = run_sliced(*c)
        if dist.get_rank() == 0:
            print(f"ep ok same_device={int(SAME_DEVICE)} world={world} schedule=coordinated L={c[-1]} case={c} "
                  f"rounds={st.a2a_rounds}+{st.allgather_rounds}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
