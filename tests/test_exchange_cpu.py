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
