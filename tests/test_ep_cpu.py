"""Expert-parallel host logic on CPU: world_size 2 and 4 over gloo.

Each rank holds a contiguous token shard; the all-gather of per-rank expert
counts, the exchange plan (global capacity, slot prefixes, send/recv splits)
and the two all-to-alls run for real over gloo with CPU tensors; the device
kernels are emulated with the oracle. Checked against the oracle run on the
concatenated batch: global slots bit-exact, received expert rows equal the
global expert buffers, combined outputs equal the single-batch combine.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_oracle as O
from paper_2201_05596_b200.ep import exchange_rows, gather_counts, make_exchange_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(world, seed):
    rng = np.random.default_rng(seed)
    S_loc, E, k, cf, M = 257, 8 * world, 2 if seed % 2 else 1, 0.8, 5
    S = S_loc * world
    logits = rng.standard_normal((S, E)) + rng.normal(0, 1.0, size=(1, E))
    x = rng.standard_normal((S, M))
    return S_loc, E, k, cf, M, logits, x


def _worker(rank, world, port, seed, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        S_loc, E, k, cf, M, logits, x = _case(world, seed)
        S = S_loc * world
        ids_all, gp_all, _ = O.top_k_gate(logits, E, k)
        g_slots, g_load, cap = O.build_dispatch_plan(ids_all, E, k, cf)
        lo, hi = rank * S_loc, (rank + 1) * S_loc
        ids, gp, xs = ids_all[lo:hi], gp_all[lo:hi], x[lo:hi]
        # local (shard) slots with unbounded capacity + per-expert counts
        local_slots, _, _ = O.build_dispatch_plan(ids, E, k, 1e9)
        totals = torch.from_numpy(np.bincount(ids.reshape(-1), minlength=E).astype(np.int32))
        counts = gather_counts(torch.empty(world * E, dtype=torch.int32), totals).numpy()
        s_total = int(counts.sum()) // k
        assert s_total == S
        assert O.capacity(E, k, cf, s_total) == cap
        plan = make_exchange_plan(counts, cap, rank, E)
        # global slots = rank prefix + local slot: bit-exact with the whole-batch plan
        gslot = plan.base[rank][ids] + local_slots
        gslot = np.where(gslot < cap, gslot, -1)
        assert np.array_equal(gslot, g_slots[lo:hi])
        # dispatch into the send layout (owner, expert, slot)
        send = torch.zeros((max(S_loc * k, 1), M), dtype=torch.float64)
        row_index = np.full((S_loc, k), -1)
        for t in range(S_loc):
            for j in range(k):
                if gslot[t, j] >= 0:
                    e = ids[t, j]
                    r = plan.send_row_base[e] + gslot[t, j] - plan.base[rank][e]
                    send[r] = torch.from_numpy(xs[t])
                    row_index[t, j] = r
        assert plan.n_send == int((row_index >= 0).sum())
        recv = torch.zeros((max(plan.n_recv, 1), M), dtype=torch.float64)
        got = exchange_rows(recv, send, plan.recv_splits, plan.send_splits)
        # received segments equal the whole-batch expert buffers in slot order
        data, occ = O.scatter_tokens(x, ids_all, g_slots, E, cap)
        e0 = rank * plan.E_loc
        for g, (st, n) in enumerate(zip(plan.seg_row_start, plan.seg_rows)):
            s, el = divmod(g, plan.E_loc)
            b = plan.base[s][e0 + el]
            assert np.array_equal(got[st:st + n].numpy(), data[e0 + el, b:b + n])
        assert np.array_equal(plan.expert_load, g_load[e0:e0 + plan.E_loc])
        # stand-in expert compute, return all-to-all, combine by row index
        y = torch.tanh(recv)
        ret = torch.zeros((max(S_loc * k, 1), M), dtype=torch.float64)
        exchange_rows(ret, y, plan.send_splits, plan.recv_splits)
        out = np.zeros((S_loc, M))
        for t in range(S_loc):
            for j in range(k):
                if row_index[t, j] >= 0:
                    out[t] += gp[t, j] * ret[row_index[t, j]].numpy()
        want = O.combine_tokens(np.tanh(data), ids_all, g_slots, gp_all)[lo:hi]
        assert np.max(np.abs(out - want), initial=0.0) <= 1e-12
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # surface the failure in the parent
        import traceback

        errq.put(f"rank {rank}: {exc!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,seed", [(2, 1), (2, 2), (4, 3)])
def test_ep_exchange_gloo(world, seed):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), "\n".join(errs)


def test_exchange_plan_properties():
    rng = np.random.default_rng(0)
    for world in (1, 2, 4, 8):
        E = 16 * world
        counts = rng.integers(0, 900, size=(world, E))
        cap = int(counts.sum(axis=0).mean())
        for r in range(world):
            p = make_exchange_plan(counts, cap, r, E)
            # every kept row is sent exactly once; per-expert totals respect capacity
            assert p.n_send == int(p.kept[r].sum())
            assert (p.kept.sum(axis=0) == np.minimum(counts.sum(axis=0), cap)).all()
            assert p.n_recv == int(p.seg_rows.sum()) == int(p.expert_load.sum())
            assert (p.expert_load <= cap).all()
    with pytest.raises(ValueError):
        make_exchange_plan(np.zeros((3, 8)), 4, 0, 8)
