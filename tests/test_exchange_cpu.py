"""The exchange schedules (paper_2201_05596_b200/exchange.py) over gloo on CPU,
pinned to the reference's own schedule simulator: tests/golden/commsim.npz holds
seeded payloads and the receive lists + trace totals that moekit.commsim
produced for them (tests/golden/make_golden.py::commsim_cases). Each rank sends
64-byte rows tagged (src, token); the rows it receives, in order, must equal
the reference's delivery, and the schedule's totals must equal the trace's."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_05596_b200.exchange import Exchanger, ScheduleError
from tests.conftest import GOLDEN

Z = np.load(os.path.join(GOLDEN, "commsim.npz"))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rows(items):
    out = torch.zeros((max(len(items), 1), 8), dtype=torch.int64)  # 64 B per item
    for i, (src, tok) in enumerate(items):
        out[i, 0], out[i, 1] = src, tok
    return out


def _worker(rank, world, port, cases, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        for case in cases:
            _check(rank, world, case)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


def _check(rank, world, case):
    if True:
        kind, _, param = (int(v) for v in Z[f"c{case}_cfg"])
        sends, send_rank = Z[f"c{case}_sends"], Z[f"c{case}_send_rank"]
        recv = Z[f"c{case}_recv"]
        mine = sends[send_rank == rank]
        order = np.argsort(mine[:, 1], kind="stable")  # send list ordered by destination
        mine = mine[order]
        want = [(int(a), int(b)) for r, a, b in recv if r == rank]
        if kind == 0:
            ex = Exchanger(schedule="hierarchical", gpus_per_node=param)
            C = np.zeros((world, world), dtype=np.int64)
            np.add.at(C, (send_rank, sends[:, 1]), 1)
            inp = _rows([(s, t) for s, _, t, _ in mine])
            out = torch.zeros((max(int(C[:, rank].sum()), 1), 8), dtype=torch.int64)
            got = ex.all_to_all(out, inp, C)
            flat = Exchanger(schedule="flat")
            got_flat = flat.all_to_all(torch.zeros_like(out), inp, C)
            assert torch.equal(got, got_flat)
            fs = flat.last_stats
            assert fs.volume_bytes == int(Z[f"c{case}_flat_volume"])
            assert fs.a2a_rounds == int(Z[f"c{case}_flat_rounds"])
        else:
            L = param
            ex = Exchanger(schedule="coordinated", tensor_slice=L)
            Q = world // L
            q = rank // L
            lead = send_rank % L == 0  # the logical payload: one replica per group
            Cg = np.zeros((Q, Q), dtype=np.int64)
            np.add.at(Cg, (send_rank[lead] // L, sends[lead, 1]), 1)
            inp = _rows([(s, t) for s, _, t, _ in mine])
            assert all(int(s) == q for s, _, _, _ in mine)
            out = torch.zeros((max(int(Cg[:, q].sum()), 1), 8), dtype=torch.int64)
            got = ex.coordinated(out, inp, Cg)
        got_l = [(int(a), int(b)) for a, b in got[:, :2].tolist()]
        assert got_l == want, (rank, got_l[:8], want[:8])
        st = ex.last_stats
        stats = [st.a2a_rounds, st.allgather_rounds, st.volume_bytes, st.a2a_volume_bytes,
                 st.reference_bytes]
        assert stats == [int(v) for v in Z[f"c{case}_stats"]], (case, stats, Z[f"c{case}_stats"])


@pytest.mark.parametrize("world", [2, 4])
def test_schedules_match_reference_commsim(world):
    cases = [c for c in range(int(Z["n"])) if int(Z[f"c{c}_cfg"][1]) == world]
    assert cases
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), "\n".join(errs)


def test_schedule_validation():
    with pytest.raises(ScheduleError):  # checked before any process-group call
        Exchanger(schedule="ring")


# ---------------------------------------------------------------------------
# C6 at scale: the schedules' index plans, with the collectives simulated in
# NumPy, for every world size 1..64 and every node size / tensor slice that
# divides it (pkg/tests/test_acceptance.py::test_c06_schedule_equivalence)
# ---------------------------------------------------------------------------

def _payload(world, per_rank, seed):
    """synthetic_sends-like payload: per rank, items with random destinations;
    rows tagged (src, token), each rank's rows ordered by destination."""
    rng = np.random.default_rng(seed)
    C = np.zeros((world, world), dtype=np.int64)
    rows, token = [], 0
    for src in range(world):
        dst = rng.integers(world, size=per_rank)
        toks = np.arange(token, token + per_rank)
        token += per_rank
        order = np.argsort(dst, kind="stable")
        rows.append(np.stack([np.full(per_rank, src), toks[order]], axis=1))
        np.add.at(C[src], dst, 1)
    return C, rows


def _split(a, sizes):
    return np.split(a, np.cumsum(sizes)[:-1]) if len(sizes) else []


def _flat(C, rows):
    world = len(rows)
    chunks = [_split(rows[s], C[s]) for s in range(world)]
    return [np.concatenate([chunks[s][d] for s in range(world)]) for d in range(world)]


def _sim_hier(C, rows, G):
    from paper_2201_05596_b200.exchange import hierarchical_plan

    world, nodes = len(rows), len(rows) // G
    pl = [hierarchical_plan(C, G, r) for r in range(world)]
    send1 = [_split(rows[r][pl[r]["idx1"]], pl[r]["in1"]) for r in range(world)]
    mid = []
    for r in range(world):
        n, l = divmod(r, G)
        m_ = np.concatenate([send1[n * G + sp][l] for sp in range(G)])
        assert len(m_) == sum(pl[r]["out1"])
        mid.append(m_)
    send2 = [_split(mid[r][pl[r]["idx2"]], pl[r]["in2"]) for r in range(world)]
    out = []
    for r in range(world):
        m, l = divmod(r, G)
        o = np.concatenate([send2[mp * G + l][m] for mp in range(nodes)])
        assert len(o) == sum(pl[r]["out2"])
        out.append(o)
    return out


def _sim_coord(Cg, rows_g, L):
    from paper_2201_05596_b200.exchange import coordinated_plan

    Q = len(rows_g)
    world = Q * L
    pl = [coordinated_plan(Cg, L, r) for r in range(world)]
    send1 = [_split(rows_g[r // L][pl[r]["idx1"]], pl[r]["in1"]) for r in range(world)]
    held = []
    for r in range(world):
        q, t = divmod(r, L)
        h = np.concatenate([send1[d * L + t][q] for d in range(Q)])  # rail t, from every group
        assert len(h) == sum(pl[r]["out1"])
        pad = np.full((pl[r]["maxh"], 2), -1, dtype=np.int64)
        pad[:len(h)] = h
        held.append(pad)
    out = []
    for r in range(world):
        q = r // L
        gathered = np.concatenate([held[q * L + u] for u in range(L)])  # all-gather in the group
        out.append(gathered[pl[r]["idx2"]])
    return out


def test_c06_schedule_plans_at_scale():
    for p in range(1, 65):
        C, rows = _payload(p, 3, seed=p)
        flat = _flat(C, rows)
        divisors = [d for d in range(1, p + 1) if p % d == 0]
        for G in divisors:
            hier = _sim_hier(C, rows, G)
            for r in range(p):
                assert np.array_equal(hier[r], flat[r]), (p, G, r)
        for L in divisors:
            Cg, rows_g = _payload(p // L, 3, seed=1000 + p)
            base = _flat(Cg, rows_g)
            coord = _sim_coord(Cg, rows_g, L)
            for r in range(p):
                assert np.array_equal(coord[r], base[r // L]), (p, L, r)
