"""All-to-all schedules for the expert-parallel exchange, on real row buffers.

The reference models three schedules as round-level simulations over
``Item`` lists (commsim.py:239-464); here they move the dispatched token rows
with NCCL (gloo for the CPU tests). Every schedule delivers the receive buffer
ordered by source rank, each source's rows in its send order - the same bytes
in the same order as the flat exchange, which is commsim's delivery contract
(recv sorted by (src, token), commsim.py:188-189, tests/test_commsim.py:85-97).

  flat          one all_to_all_single (commsim.py:239-277: p pairwise rounds).
  hierarchical  (commsim.py:280-370) two phases for ranks grouped G per node:
                regroup rows by the destination's local id (layout transform),
                all-to-all inside the node, regroup by destination node, then
                all-to-all between the same-local-id ranks of all nodes (the
                "rail"). G + p/G rounds, every byte moves twice.
  coordinated   (commsim.py:373-464) for tensor-sliced groups of L consecutive
                ranks holding identical copies of their group's payload:
                replica t sends only the rows at positions i = t (mod L) of
                each destination block to replica t of the destination group
                (p/L rounds, payload moved once), then an all-gather inside
                each group rebuilds the full receive set on every member.

Counts are host integers (the EP layer already syncs its all-gathered expert
counts for the NCCL splits). Layout transforms are row permutations:
``moe_gather_rows`` on the GPU. The CPU branch in ``_gather`` exists only so
the gloo tests can drive this host logic without a GPU; device tensors never
take it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["ScheduleError", "ReplicaMismatchError", "ExchangeStats", "Exchanger",
           "hierarchical_plan", "coordinated_plan", "device_collectives", "all_gather_flat",
           "all_reduce_sum"]


class ScheduleError(ValueError):
    """Impossible schedule parameters (commsim.py:62-63)."""


class ReplicaMismatchError(ScheduleError):
    """Ranks that should hold identical replicas disagree (commsim.py:66-67)."""


@dataclass(frozen=True)
class ExchangeStats:
    """The CommTrace totals (commsim.py:108-140) of one exchange, global over ranks."""

    schedule: str
    world_size: int
    a2a_rounds: int
    allgather_rounds: int
    volume_bytes: int
    a2a_volume_bytes: int
    reference_bytes: int

    @property
    def rounds(self) -> int:
        return self.a2a_rounds + self.allgather_rounds

    @property
    def volume_ratio(self) -> float:
        return self.volume_bytes / self.reference_bytes if self.reference_bytes else 0.0


def _ranges(starts, lens) -> np.ndarray:
    """Concatenation of arange(s, s + n) over (starts, lens)."""
    starts = np.asarray(starts, dtype=np.int64).reshape(-1)
    lens = np.asarray(lens, dtype=np.int64).reshape(-1)
    tot = int(lens.sum())
    if tot == 0:
        return np.zeros(0, dtype=np.int64)
    shift = starts - np.concatenate([[0], np.cumsum(lens)[:-1]])
    return np.repeat(shift, lens) + np.arange(tot, dtype=np.int64)


def _excl(a, axis=-1) -> np.ndarray:
    a = np.asarray(a, dtype=np.int64)
    c = np.cumsum(a, axis=axis)
    return c - a


def _gather(dst: torch.Tensor, src: torch.Tensor, idx: np.ndarray) -> torch.Tensor:
    """dst[:n] = src[idx] (one layout transform)."""
    n = int(idx.size)
    if n == 0:
        return dst[:0]
    if src.is_cuda:
        it = torch.from_numpy(idx.astype(np.int32)).to(src.device, non_blocking=True)
        _lib.call("moe_gather_rows", src.data_ptr(), src.shape[1] * src.element_size(),
                  it.data_ptr(), n, dst.data_ptr(), _lib.stream_ptr())
    else:  # gloo tests of the host logic only
        torch.index_select(src, 0, torch.from_numpy(idx.astype(np.int64)), out=dst[:n])
    return dst[:n]


def device_collectives(group=None) -> bool:
    """NCCL groups move device tensors directly. Gloo groups move host tensors:
    the CPU tests, and several ranks sharing ONE GPU (NCCL refuses duplicate
    devices; the single-GPU EP parity test runs that way) - device tensors
    are staged through host memory there."""
    return dist.get_backend(group) == "nccl"


def _staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and not device_collectives(group)


def all_gather_flat(out: torch.Tensor, inp: torch.Tensor, group=None) -> torch.Tensor:
    """out[r*n:(r+1)*n] = inp of rank r (out is (world*n, ...) contiguous)."""
    if _staged(inp, group):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)
    return out


def all_reduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)
    return t


def _a2a(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group) -> torch.Tensor:
    n_out, n_in = int(sum(out_splits)), int(sum(in_splits))
    osz, isz = [int(v) for v in out_splits], [int(v) for v in in_splits]
    if _staged(inp, group):
        o = torch.empty((n_out,) + tuple(out.shape[1:]), dtype=out.dtype)
        dist.all_to_all_single(o, inp[:n_in].cpu(), output_split_sizes=osz, input_split_sizes=isz,
                               group=group)
        out[:n_out].copy_(o)
    else:
        dist.all_to_all_single(out[:n_out], inp[:n_in], output_split_sizes=osz,
                               input_split_sizes=isz, group=group)
    return out[:n_out]


def hierarchical_plan(C, G: int, r: int) -> dict:
    """Rank r's side of the two-phase schedule (pure index arithmetic).

    C[s][d]: rows s sends to d, ranks node-major in nodes of G. Phase 1 sends
    ``inp[idx1]`` split ``in1`` to the node's local ids and receives ``out1``
    from them ([source local id][destination node] blocks); phase 2 sends
    ``mid[idx2]`` split ``in2`` along the rail (destination nodes) and receives
    ``out2``, ordered by global source rank."""
    C = np.asarray(C, dtype=np.int64)
    world = C.shape[0]
    nodes = world // G
    n, l = divmod(r, G)
    off = _excl(C[r])
    d_order = np.array([m * G + lp for lp in range(G) for m in range(nodes)], dtype=np.int64)
    idx1 = _ranges(off[d_order], C[r][d_order])
    in1 = [int(C[r][lp::G].sum()) for lp in range(G)]
    out1 = [int(C[n * G + sp][l::G].sum()) for sp in range(G)]
    blk = np.array([[C[n * G + sp][m * G + l] for m in range(nodes)] for sp in range(G)],
                   dtype=np.int64).reshape(G, nodes)
    boff = _excl(blk.reshape(-1)).reshape(G, nodes)
    idx2 = _ranges(boff.T.reshape(-1), blk.T.reshape(-1))
    in2 = [int(blk[:, m].sum()) for m in range(nodes)]
    out2 = [int(C[mp * G:(mp + 1) * G, r].sum()) for mp in range(nodes)]
    return dict(idx1=idx1, in1=in1, out1=out1, idx2=idx2, in2=in2, out2=out2)


def coordinated_plan(Cg, L: int, rank: int) -> dict:
    """Rank's side of the coordinated schedule (pure index arithmetic).

    Cg[q][D]: logical rows group q sends to group D. The rail exchange sends
    ``inp[idx1]`` (positions = t mod L of each destination block) split
    ``in1`` and receives ``out1`` into a buffer of ``maxh`` rows; after the
    all-gather inside the group (L x maxh rows, member-major) the group's
    receive list is ``gathered[idx2]``."""
    Cg = np.asarray(Cg, dtype=np.int64)
    Q = Cg.shape[0]
    q, t = divmod(rank, L)

    def share(c, u):  # rows i < c with i = u (mod L)
        return np.maximum(0, (np.asarray(c, dtype=np.int64) - u + L - 1) // L)

    off = _excl(Cg[q])
    cnt = share(Cg[q], t)
    idx1 = _ranges(off + t, cnt)
    if L > 1 and idx1.size:  # positions t + L*j inside each block
        base = np.repeat(off + t, cnt)
        idx1 = base + (idx1 - base) * L
    hu = np.stack([share(Cg[:, q], u) for u in range(L)]).reshape(L, Q)  # rows per member
    maxh = max(int(hu.sum(axis=1).max()), 1)
    huo = _excl(hu, axis=1)
    parts = []
    for qs in range(Q):
        i = np.arange(int(Cg[qs, q]), dtype=np.int64)
        u = i % L
        parts.append(u * maxh + huo[u, qs] + i // L)
    idx2 = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    held = np.array([[int(share(Cg[:, qq], u).sum()) for u in range(L)] for qq in range(Q)])
    return dict(idx1=idx1, in1=[int(v) for v in cnt], out1=[int(v) for v in share(Cg[:, q], t)],
                maxh=maxh, idx2=idx2, allgather_rows=int(held.sum()) * (L - 1))


class Exchanger:
    """One schedule bound to a process group (subgroups are created here, so
    every rank of ``group`` must construct it, in the same order)."""

    def __init__(self, group=None, schedule: str = "flat", gpus_per_node: int | None = None,
                 tensor_slice: int = 1) -> None:
        if schedule not in ("flat", "hierarchical", "coordinated"):
            raise ScheduleError(f"unknown schedule {schedule!r}")
        self.group, self.schedule = group, schedule
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        ranks = dist.get_process_group_ranks(group) if group is not None else list(range(self.world))
        self._scratch: dict = {}
        self.last_stats: ExchangeStats | None = None
        if schedule == "hierarchical":
            G = int(gpus_per_node or 0)
            if G < 1 or self.world % G:
                raise ScheduleError(f"gpus_per_node {gpus_per_node} must divide world {self.world}")
            self.G, self.nodes = G, self.world // G
            self.node_group = self.rail_group = None
            for n in range(self.nodes):  # node n: ranks n*G .. n*G+G-1 (node-major numbering)
                g = dist.new_group([ranks[n * G + l] for l in range(G)])
                if self.rank // G == n:
                    self.node_group = g
            for l in range(G):  # rail l: the local-id-l rank of every node
                g = dist.new_group([ranks[m * G + l] for m in range(self.nodes)])
                if self.rank % G == l:
                    self.rail_group = g
        if schedule == "coordinated":
            L = int(tensor_slice)
            if L < 1 or self.world % L:
                raise ScheduleError(f"tensor_slice {tensor_slice} must divide world {self.world}")
            self.L, self.Q = L, self.world // L
            self.slice_group = self.rail_group = None
            for q in range(self.Q):  # tensor group q: ranks q*L .. q*L+L-1
                g = dist.new_group([ranks[q * L + u] for u in range(L)])
                if self.rank // L == q:
                    self.slice_group = g
            for t in range(L):  # replica rail t: member t of every group
                g = dist.new_group([ranks[d * L + t] for d in range(self.Q)])
                if self.rank % L == t:
                    self.rail_group = g

    # ------------------------------------------------------------------
    def _buf(self, name: str, rows: int, like: torch.Tensor) -> torch.Tensor:
        b = self._scratch.get(name)
        if b is None or b.shape[0] < rows or b.shape[1:] != like.shape[1:] or b.dtype != like.dtype \
                or b.device != like.device:
            b = torch.empty((max(rows, 1),) + tuple(like.shape[1:]), dtype=like.dtype,
                            device=like.device)
            self._scratch[name] = b
        return b

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, counts) -> torch.Tensor:
        """counts[s][d] = rows rank s sends to rank d (identical on every rank).
        ``inp`` holds this rank's rows ordered by destination; returns the
        received rows ordered by source (a view of ``out``)."""
        if self.schedule == "coordinated":
            raise ScheduleError("use coordinated() for the coordinated schedule")
        C = np.asarray(counts, dtype=np.int64)
        if C.shape != (self.world, self.world):
            raise ScheduleError(f"counts shape {C.shape} != ({self.world}, {self.world})")
        r = self.rank
        row_bytes = int(inp.shape[1] * inp.element_size()) if inp.dim() == 2 else inp.element_size()
        payload = int(C.sum()) * row_bytes
        if self.schedule == "flat" or self.world == 1:
            self.last_stats = ExchangeStats("flat", self.world, self.world, 0, payload, payload,
                                            payload)
            return _a2a(out, inp, C[:, r], C[r], self.group)
        G, nodes = self.G, self.nodes
        pl = hierarchical_plan(C, G, r)
        send1 = _gather(self._buf("send1", int(C[r].sum()), inp), inp, pl["idx1"])
        mid = _a2a(self._buf("mid", sum(pl["out1"]), inp), send1, pl["out1"], pl["in1"],
                   self.node_group)
        send2 = _gather(self._buf("send2", pl["idx2"].size, inp), mid, pl["idx2"])
        out2, in2 = pl["out2"], pl["in2"]
        # received: [source node m'][source local id s'] = ordered by global source rank
        res = _a2a(out, send2, out2, in2, self.rail_group)
        self.last_stats = ExchangeStats("hierarchical", self.world, G + nodes, 0, 2 * payload,
                                        2 * payload, payload)
        return res

    def coordinated(self, out: torch.Tensor, inp: torch.Tensor, group_counts) -> torch.Tensor:
        """group_counts[q][D] = rows logical group q sends to group D. ``inp`` is
        this rank's group send list ordered by destination group (every member
        of a group holds the same list); returns the group's receive list ordered
        by source group, identical on every member."""
        if self.schedule != "coordinated":
            raise ScheduleError("coordinated() needs schedule='coordinated'")
        Cg = np.asarray(group_counts, dtype=np.int64)
        L, Q = self.L, self.Q
        if Cg.shape != (Q, Q):
            raise ScheduleError(f"group counts shape {Cg.shape} != ({Q}, {Q})")
        row_bytes = int(inp.shape[1] * inp.element_size())
        pl = coordinated_plan(Cg, L, self.rank)
        send1 = _gather(self._buf("send1", pl["idx1"].size, inp), inp, pl["idx1"])
        # the rail exchange lands in a buffer padded to the largest member's share,
        # which is then all-gathered inside the tensor group
        maxh = pl["maxh"]
        pad = self._buf("pad", maxh, inp)
        _a2a(pad, send1, pl["out1"], pl["in1"], self.rail_group)
        gbuf = self._buf("gath", L * maxh, inp)[:L * maxh]
        if L > 1:
            all_gather_flat(gbuf, pad[:maxh], group=self.slice_group)
        else:
            gbuf = pad[:maxh]
        # reassemble each source block: position i came from member i % L
        res = _gather(out, gbuf, pl["idx2"])
        payload = int(Cg.sum()) * row_bytes
        # all-gather volume: each member's share to its L-1 peers (commsim.py:440-455)
        ag = pl["allgather_rows"] * row_bytes
        self.last_stats = ExchangeStats("coordinated", self.world, Q, L, payload + ag, payload,
                                        payload)
        return res
