"""Expert parallelism for the MoE layer across the GPUs of one NVSwitch box.

Partitioning: rank r holds a contiguous block of tokens and
the contiguous expert block [r*E/p, (r+1)*E/p) (planner.py:101-109, with
E % p == 0 as planner.py:202-206 requires). The gate (and the Residual-MoE
shared MLP) is replicated.

Capacity is GLOBAL: cap = ceil(cf * S_total * k / E), and slots are counted
over the whole batch in token-major order. Because token-major order over the
concatenated batch equals rank-major order over contiguous shards, a token's
global slot = (assignments to its expert on lower ranks) + (its slot within
its own shard). One all-gather of the per-rank (E,) expert counts gives every
rank those prefixes, so routing, slots and the dropped set are bit-identical
to ``build_dispatch_plan`` run on the whole batch at any p.

Two transports. "p2p" (default for the flat schedule, every layer kind): no
collective on the data path - the counts are all-gathered over peer memory,
the plan is computed on device (no host sync), the dispatch kernel stores each
kept row straight into its owner's receive buffer over NVLink (laid out
[local expert][global slot], i.e. the single-GPU expert buffer), and the
owner's GEMM2 epilogue stores every row straight back to its source: k=1
layers combined (x + p*y) into the source's output slot, k=2 / Residual-MoE
expert rows into the source's return buffer, which the source combines
locally (plus its replicated shared MLP). System-scope flag barriers separate
the phases. (chunks > 1: the round-1 pipelined variant, owner-local combine
and a source-side pull.)

"nccl" (any k, shared MLP; the hierarchical schedule) - one all-to-all each way, flat (one NCCL
all_to_all_single) or, with schedule="hierarchical", the two-phase
node/rail schedule of commsim.py:280-370 (exchange.py):
  send buffer on rank r : kept rows ordered (owner rank, expert, slot)
  receive buffer        : [source rank][local expert][rows in slot order]
                          (commsim's delivery contract: ordered by source,
                          commsim.py:188-189, flat schedule :239-277)
  the grouped GEMM runs directly on the receive layout (one group per
  (source, local expert) segment), the results go back with the inverse
  all-to-all, and the combine gathers them by the row index dispatch wrote.

``SlicedEPMoeLayer``: tensor-sliced groups of L ranks (planner tensor_slice,
planner.py:160-174) that hold identical token shards; experts are block-sharded
over the groups and each expert's FFN is sliced L ways along d_ff inside its
group (expert slicing, planner.py:207-222 - with one expert per group this is
the planner's latency mode for p > E). Tokens move with the coordinated
schedule (commsim.py:373-464), the slices' partial GEMM2 outputs are summed
with an all-reduce inside the group, and every member combines its group's
tokens.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .arch import FFN_MULT, DenseFfn, LayerSpec, MoeLayerParams, _Phases, _t
from .exchange import Exchanger, ReplicaMismatchError, _a2a, all_gather_flat, all_reduce_sum
from .gating import GatingConfig
from .tensor import ShapeError

__all__ = ["ExchangePlan", "make_exchange_plan", "gather_counts", "exchange_rows", "EPMoeLayer",
           "SlicedEPMoeLayer", "rank_counts"]


@dataclass
class ExchangePlan:
    world: int
    rank: int
    E: int
    E_loc: int
    cap: int
    counts: np.ndarray          # (world, E) assignments per rank and expert (before drops)
    base: np.ndarray            # (world, E) global slot of each rank's first assignment to e
    kept: np.ndarray            # (world, E) kept assignments per rank and expert
    send_row_base: np.ndarray   # (E,) this rank's send-buffer start row per expert
    send_splits: list           # rows to each destination rank
    recv_splits: list           # rows from each source rank
    seg_row_start: np.ndarray   # (world*E_loc,) receive-buffer start of (src, local expert)
    seg_rows: np.ndarray        # (world*E_loc,)
    seg_weight: np.ndarray      # (world*E_loc,) local expert index
    expert_load: np.ndarray     # (E_loc,) kept rows per local expert (= min(total, cap))

    @property
    def n_send(self) -> int:
        return int(sum(self.send_splits))

    @property
    def n_recv(self) -> int:
        return int(sum(self.recv_splits))


def make_exchange_plan(counts: np.ndarray, cap: int, rank: int, num_experts: int) -> ExchangePlan:
    """Host-side split arithmetic from the all-gathered (world, E) counts."""
    counts = np.asarray(counts, dtype=np.int64)
    world, E = counts.shape
    if E != num_experts or E % world:
        raise ValueError(f"E={E} must equal num_experts and divide evenly over {world} ranks")
    e_loc = E // world
    base = np.zeros_like(counts)
    base[1:] = np.cumsum(counts, axis=0)[:-1]
    kept = np.clip(cap - base, 0, counts)
    mine = kept[rank]
    send_row_base = np.zeros(E, dtype=np.int64)
    send_row_base[1:] = np.cumsum(mine)[:-1]
    send_splits = [int(mine[o * e_loc:(o + 1) * e_loc].sum()) for o in range(world)]
    lo, hi = rank * e_loc, (rank + 1) * e_loc
    recv_splits = [int(kept[s, lo:hi].sum()) for s in range(world)]
    seg_rows = kept[:, lo:hi].reshape(-1)
    seg_row_start = np.zeros_like(seg_rows)
    seg_row_start[1:] = np.cumsum(seg_rows)[:-1]
    seg_weight = np.tile(np.arange(e_loc), world)
    expert_load = np.minimum(counts[:, lo:hi].sum(axis=0), cap)
    assert int(expert_load.sum()) == int(seg_rows.sum())
    return ExchangePlan(world=world, rank=rank, E=E, E_loc=e_loc, cap=cap, counts=counts,
                        base=base, kept=kept, send_row_base=send_row_base,
                        send_splits=send_splits, recv_splits=recv_splits,
                        seg_row_start=seg_row_start, seg_rows=seg_rows, seg_weight=seg_weight,
                        expert_load=expert_load)


def rank_counts(plan: ExchangePlan) -> np.ndarray:
    """(world, world) kept rows source rank -> owner rank (the exchange's split matrix)."""
    return plan.kept.reshape(plan.world, plan.world, plan.E_loc).sum(axis=2)


def gather_counts(out_flat: torch.Tensor, totals: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's (E,) expert counts into a flat (world*E,) tensor."""
    all_gather_flat(out_flat, totals, group=group)
    return out_flat.view(-1, totals.numel())


def exchange_rows(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group=None):
    """One flat all-to-all of variable row counts (NCCL on GPU, gloo on CPU)."""
    return _a2a(out, inp, out_splits, in_splits, group)


class EPMoeLayer:
    """One MoE layer sharded over the ranks of ``group`` (bf16, tcgen05 path)."""

    def __init__(self, spec: LayerSpec, gate_w, local_experts, shared=None, group=None,
                 dtype=torch.bfloat16, device=None, transport: str = "auto",
                 schedule: str = "flat", gpus_per_node: int | None = None, chunks: int = 1,
                 comm_sms: int = 16) -> None:
        if spec.kind != "moe":
            raise ShapeError("EPMoeLayer needs a moe LayerSpec")
        if dtype != torch.bfloat16:
            raise TypeError("the expert-parallel path is bf16 (tcgen05)")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        E, M = spec.experts, spec.hidden
        if E % self.world:
            raise ValueError(f"{E} experts do not divide over {self.world} ranks (planner.py:202-206)")
        dev = _lib.require_device(None) if device is None else torch.device(device)
        self.spec, self.dev, self.dtype = spec, dev, dtype
        self.E, self.M, self.F, self.k = E, M, FFN_MULT * M, spec.gating.k
        self.E_loc = E // self.world
        if len(local_experts) != self.E_loc:
            raise ShapeError(f"{len(local_experts)} local experts, expected {self.E_loc}")
        gw = _t(gate_w, dev, torch.float32)
        self.epad = max(32, 1 << (E - 1).bit_length())
        self.wg = torch.zeros((self.epad, M), dtype=torch.bfloat16, device=dev)
        self.wg[:E] = gw.t().to(torch.bfloat16)
        F = self.F
        self.w1 = torch.empty((self.E_loc * F, M), dtype=torch.bfloat16, device=dev)
        self.w2 = torch.empty((self.E_loc * M, F), dtype=torch.bfloat16, device=dev)
        self.b1 = torch.empty((self.E_loc, F), dtype=torch.float32, device=dev)
        self.b2 = torch.empty((self.E_loc, M), dtype=torch.float32, device=dev)
        for i, p in enumerate(local_experts):  # one expert at a time: bounded peak memory
            self.w1[i * F:(i + 1) * F] = _t(p.w1, dev, torch.bfloat16).t()
            self.w2[i * M:(i + 1) * M] = _t(p.w2, dev, torch.bfloat16).t()
            self.b1[i] = _t(p.b1, dev, torch.float32).reshape(F)
            self.b2[i] = _t(p.b2, dev, torch.float32).reshape(M)
        self.shared = DenseFfn(shared, M, dtype, dev) if spec.residual else None
        # "p2p": dispatch stores rows into the owners' receive buffers and the owners'
        # GEMM2 epilogue stores every row straight back into its source (combined
        # into the output for k=1 layers; expert outputs into a return buffer that
        # the source combines locally for k=2 / Residual-MoE), over NVLink peer
        # memory; "nccl": two all_to_all_single exchanges.
        if transport == "auto":
            transport = "p2p" if schedule == "flat" else "nccl"
        if schedule != "flat" and transport != "nccl":
            raise ValueError(f"schedule {schedule!r} runs on the nccl transport")
        if transport not in ("p2p", "nccl"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        self.schedule = schedule
        # p2p only: split every rank's tokens into `chunks` so chunk c+1's dispatch and
        # chunk c-1's return pull run beside chunk c's GEMMs (on `comm_sms` SMs the
        # GEMMs leave free, from a second stream)
        if chunks < 1 or (chunks > 1 and transport != "p2p"):
            raise ValueError("chunks > 1 needs the p2p transport")
        if chunks > 1 and (self.k != 1 or self.shared is not None):
            raise ValueError("the chunked p2p pipeline covers k=1 layers without a shared MLP")
        self.chunks, self.comm_sms = int(chunks), int(comm_sms)
        self.exchanger = Exchanger(group, schedule, gpus_per_node) if transport == "nccl" else None
        self._ws: dict = {}
        self._p2p: dict | None = None
        self._pipe = None
        self.last_plan: ExchangePlan | None = None

    @classmethod
    def from_params(cls, spec: LayerSpec, params: MoeLayerParams, group=None, **kw):
        """Take this rank's expert block out of full (replicated) parameters."""
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        e_loc = spec.experts // world
        local = params.experts[rank * e_loc:(rank + 1) * e_loc]
        return cls(spec, params.gate_w, local, params.shared, group=group, **kw)

    @classmethod
    def synthetic(cls, S: int, M: int, E: int, k: int, cf: float, dev, seed: int = 0, group=None,
                  residual: bool = False, **kw):
        """Random-init layer of the named shape (N(0,1)*0.1 weights, zero biases,
        arch.py:347-365), generated on device per expert so every rank draws
        the same gate and its own expert block."""
        from .arch import FfnParams

        spec = LayerSpec(kind="moe", hidden=M, experts=E, residual=residual,
                         gating=GatingConfig(E, k, cf))
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        e_loc = E // world
        g = torch.Generator(device=dev).manual_seed(seed)
        gate_w = torch.randn(M, E, device=dev, generator=g) * 0.1
        F = FFN_MULT * M
        experts = []
        zb1, zb2 = torch.zeros(1, F, device=dev), torch.zeros(1, M, device=dev)
        for e in range(rank * e_loc, (rank + 1) * e_loc):
            ge = torch.Generator(device=dev).manual_seed(seed * 100003 + e + 1)
            w1 = torch.randn(M, F, device=dev, generator=ge, dtype=torch.bfloat16) * 0.1
            w2 = torch.randn(F, M, device=dev, generator=ge, dtype=torch.bfloat16) * 0.1
            experts.append(FfnParams(w1, zb1, w2, zb2))
        shared = None
        if residual:  # replicated: same draw on every rank
            gs = torch.Generator(device=dev).manual_seed(seed * 100003 + E + 1)
            shared = FfnParams(torch.randn(M, F, device=dev, generator=gs, dtype=torch.bfloat16) * 0.1,
                               zb1, torch.randn(F, M, device=dev, generator=gs,
                                                dtype=torch.bfloat16) * 0.1, zb2)
        return cls(spec, gate_w, experts, shared, group=group, device=dev, **kw)

    # ------------------------------------------------------------------
    def _workspace(self, S: int) -> dict:
        ws = self._ws.get(S)
        if ws is not None:
            return ws
        if len(self._ws) >= 6:
            self._ws.pop(next(iter(self._ws)))
        dev, E, M, F, k = self.dev, self.E, self.M, self.F, self.k
        T = (S + _lib.ROUTE_TILE - 1) // _lib.ROUTE_TILE
        i32 = dict(dtype=torch.int32, device=dev)
        ws = dict(
            T=T, ids=torch.empty((S, k), **i32), slots=torch.empty((S, k), **i32),
            row_index=torch.empty((S, k), **i32), local_rank=torch.empty((S, k), **i32),
            gp=torch.empty((S, k), dtype=torch.float32, device=dev),
            tile_counts=torch.empty((max(T, 1), E), **i32),
            tile_offsets=torch.empty((max(T, 1), E), **i32),
            totals=torch.empty(E, **i32), kept=torch.empty(E, **i32),
            counts=torch.empty(self.world * E, **i32),
            send=torch.empty((max(S * k, 1), M), dtype=self.dtype, device=dev),
            ret=torch.empty((max(S * k, 1), M), dtype=self.dtype, device=dev),
        )
        if self.shared is not None:
            ws["hs"] = torch.empty((max(S, 1), F), dtype=self.dtype, device=dev)
            ws["sh_rows"] = torch.tensor([S], **i32)
            ws["sh_w"] = torch.zeros(1, **i32)
        self._ws[S] = ws
        return ws

    def _recv_buffers(self, ws: dict, rows: int) -> None:
        if ws.get("recv_rows", -1) >= rows:
            return
        rows = max(rows, 1)
        ws["recv"] = torch.empty((rows, self.M), dtype=self.dtype, device=self.dev)
        ws["h"] = torch.empty((rows, self.F), dtype=self.dtype, device=self.dev)
        ws["y"] = torch.empty((rows, self.M), dtype=self.dtype, device=self.dev)
        ws["recv_rows"] = rows

    def __call__(self, x, out=None, timer=None):
        return self.forward(x, out, timer)

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, timer=None):
        """out = x + combine(experts(dispatch(x))) [+ shared(x)] for this rank's
        tokens, experts evaluated on their owner ranks. Host inputs stream
        through ``pipeline.HostPipeline`` like ``MoeLayer``."""
        if not x.is_cuda:
            if self._pipe is None:
                from .pipeline import HostPipeline

                self._pipe = HostPipeline(self._forward_dev, self.M, self.dtype, self.dev)
            oh = out if (out is not None and not out.is_cuda) else None
            return self._pipe(x.to(self.dtype), oh, timer=timer)
        return self._forward_dev(x, out, timer)

    def _forward_dev(self, x: torch.Tensor, out: torch.Tensor | None = None, timer=None):
        if self.transport == "p2p":
            return self._forward_p2p(x, out, timer)
        if x.device != self.dev:
            x = x.to(self.dev, non_blocking=True)
        x = x.to(self.dtype).contiguous()
        if x.dim() != 2 or x.shape[1] != self.M:
            raise ShapeError(f"batch width {tuple(x.shape)} does not match layer hidden {self.M}")
        S = x.shape[0]
        out = torch.empty_like(x) if out is None else out
        ws = self._workspace(S)
        E, M, F, k = self.E, self.M, self.F, self.k
        st = _lib.stream_ptr()
        ph = _Phases(timer)
        ids, gp, lr, tc = ws["ids"], ws["gp"], ws["local_rank"], ws["tile_counts"]
        ph("gate")
        if S:
            _lib.call("moe_gate_gemm_bf16", x.data_ptr(), self.wg.data_ptr(), S, M, E, k, None,
                      ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), st)
        ph("scan")
        # local per-expert counts (cap irrelevant here)
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, 2 ** 62, None,
                  ws["tile_offsets"].data_ptr(), ws["totals"].data_ptr(), ws["kept"].data_ptr(),
                  st)
        ph("counts_allgather")
        counts = gather_counts(ws["counts"], ws["totals"], self.group)
        counts = counts.cpu().numpy()  # the one host sync: splits for NCCL
        s_total = int(counts.sum()) // k
        cap = self.spec.gating.capacity(s_total)
        plan = make_exchange_plan(counts, cap, self.rank, E)
        self.last_plan = plan
        ph("scan")
        tables = np.concatenate([plan.base[self.rank], plan.send_row_base, plan.seg_row_start,
                                 plan.seg_rows, plan.seg_weight]).astype(np.int32)
        tab = torch.from_numpy(tables).to(self.dev, non_blocking=True)
        base_d, row_base_d = tab[:E], tab[E:2 * E]
        G = self.world * self.E_loc
        seg_start_d, seg_rows_d, seg_w_d = tab[2 * E:2 * E + G], tab[2 * E + G:2 * E + 2 * G], \
            tab[2 * E + 2 * G:2 * E + 3 * G]
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, cap, base_d.data_ptr(),
                  ws["tile_offsets"].data_ptr(), ws["totals"].data_ptr(), ws["kept"].data_ptr(),
                  st)
        ph("dispatch")
        if S:
            _lib.call("moe_dispatch_ep", x.data_ptr(), S, M * 2, E, k, cap, ids.data_ptr(),
                      lr.data_ptr(), ws["tile_offsets"].data_ptr(), base_d.data_ptr(),
                      row_base_d.data_ptr(), ws["slots"].data_ptr(), ws["row_index"].data_ptr(),
                      ws["send"].data_ptr(), st)
        ph("all_to_all_dispatch")
        self._recv_buffers(ws, plan.n_recv)
        C = rank_counts(plan)
        recv = self.exchanger.all_to_all(ws["recv"], ws["send"], C)
        n_recv = plan.n_recv
        max_rows = int(plan.seg_rows.max()) if plan.seg_rows.size else 0
        if n_recv and max_rows:
            ph("gemm1")
            _lib.call("moe_grouped_gemm_bf16", recv.data_ptr(), n_recv, M, self.w1.data_ptr(),
                      self.E_loc * F, F, self.b1.data_ptr(), ws["h"].data_ptr(), G,
                      seg_start_d.data_ptr(), 0, seg_rows_d.data_ptr(), 0, seg_w_d.data_ptr(),
                      max_rows, _lib.MOE_ACT_GELU, st)
            ph("gemm2")
            _lib.call("moe_grouped_gemm_bf16", ws["h"].data_ptr(), n_recv, F, self.w2.data_ptr(),
                      self.E_loc * M, M, self.b2.data_ptr(), ws["y"].data_ptr(), G,
                      seg_start_d.data_ptr(), 0, seg_rows_d.data_ptr(), 0, seg_w_d.data_ptr(),
                      max_rows, _lib.MOE_ACT_NONE, st)
        ph("all_to_all_return")
        self.exchanger.all_to_all(ws["ret"], ws["y"], C.T)
        if self.shared is not None and S:
            # shared MLP GEMM1, then GEMM2 with the combine + residual adds in its
            # epilogue, reading the returned rows (the single-GPU arithmetic)
            ph("shared_mlp")
            sh = self.shared
            _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), S, M, sh.w1.data_ptr(), F, F,
                      sh.b1.data_ptr(), ws["hs"].data_ptr(), 1, None, 0, None, S, None, S,
                      _lib.MOE_ACT_GELU | _lib.MOE_GEMM_PAD_SCRATCH, st)
            _lib.call("moe_residual_gemm_bf16", ws["hs"].data_ptr(), S, None, 0, 0, F,
                      sh.w2.data_ptr(), M, M, sh.b2.data_ptr(), ws["ret"].data_ptr(), 1, S,
                      ws["sh_rows"].data_ptr(), ws["sh_w"].data_ptr(), S, 0, 0, ids.data_ptr(),
                      None, gp.data_ptr(), k, cap, x.data_ptr(), out.data_ptr(), S,
                      ws["row_index"].data_ptr(), st)
            ph(None)
            return out
        ph("combine")
        if S:
            _lib.call("moe_combine", ws["ret"].data_ptr(), _lib.MOE_BF16, S, M, E, k, cap,
                      ids.data_ptr(), ws["slots"].data_ptr(), ws["row_index"].data_ptr(),
                      gp.data_ptr(), _lib.MOE_F32, x.data_ptr(), None, out.data_ptr(), 1, st)
        ph(None)
        return out

    def graphed(self, S: int):
        """Forward for S local tokens as one CUDA graph (all ranks must capture
        and replay in the same order)."""
        from .pipeline import GraphedForward

        return GraphedForward(self, S, self.M, self.dtype, self.dev)

    def kept_assignments(self, S: int) -> int:
        if self.transport == "p2p":
            self.check_errors()  # syncs anyway: surface a timed-out peer barrier here
            if self.chunks > 1:
                return int(self._p2p[S]["kept_c"].sum().item())
            return int(self._ws[S]["kept"].sum().item())
        return int(self.last_plan.kept[self.rank].sum()) if self.last_plan is not None else 0

    # ------------------------------------------------------------------ p2p
    def _p2p_state(self, S: int) -> dict:
        """Peer-memory layout for batch size S (cached per S; collective on first use)."""
        if self._p2p is None:
            self._p2p = {}
        st = self._p2p.get(S)
        if st is not None:
            return st
        # the peer-memory layout is sized from the global batch: all ranks equal S
        sizes = torch.tensor([S], dtype=torch.int64, device=self.dev)
        alls = torch.empty(self.world, dtype=torch.int64, device=self.dev)
        all_gather_flat(alls, sizes, group=self.group)
        if int(alls.min()) != int(alls.max()):
            raise ValueError("the peer-memory transport needs the same token count on every rank")
        from .ipc import IpcRegion

        if not hasattr(self, "_epoch_dev"):  # one barrier epoch per layer, shared by all S
            self._epoch_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self._epoch2_dev = torch.zeros(1, dtype=torch.int32, device=self.dev)

        M, k = self.M, self.k
        cap = self.spec.gating.capacity(S * self.world)
        rmax = max(self.E_loc * cap, 1)

        def al(n):
            return (n + 255) // 256 * 256

        C = self.chunks
        # push return: k=1 layers without a shared MLP get two alternating output
        # slots the owners store combined rows into; others an (S*k)-row return buffer
        push1 = k == 1 and self.shared is None
        off_recv = 0
        off_tok = off_recv + al(rmax * M * 2)
        off_prob = off_tok + al(rmax * 4)
        off_src = off_prob + al(rmax * 4)
        off_ret = off_src + al(rmax * 4)  # owner-local combined rows (chunked pull path)
        off_cnt = off_ret + (al(rmax * M * 2) if C > 1 else 0)
        off_sig = off_cnt + al(self.world * C * self.E * 4)
        off_sig2 = off_sig + al(64 * 4)  # second barrier channel (the comm stream)
        off_back = off_sig2 + al(64 * 4)  # output slots (push1) / return buffer
        back_rows = 2 * S if push1 else S * k
        total = off_back + al(max(back_rows, 1) * M * 2)
        region = IpcRegion(total, self.group, self.dev)
        i32 = dict(dtype=torch.int32, device=self.dev)
        G = self.E_loc
        st = dict(
            S=S, cap=cap, rmax=rmax, region=region,
            recv=region.tensor(off_recv, (rmax, M), torch.bfloat16),
            row_token=region.tensor(off_tok, (rmax,), torch.int32),
            row_prob=region.tensor(off_prob, (rmax,), torch.float32),
            ret=region.tensor(off_ret, (rmax, M), torch.bfloat16) if C > 1 else None,
            row_src=region.tensor(off_src, (rmax,), torch.int32), peer_src=region.ptr_table(off_src),
            push1=push1,
            oslot=[region.tensor(off_back + i * S * M * 2, (S, M), torch.bfloat16)
                   for i in range(2)] if push1 else None,
            peer_oslot=[region.ptr_table(off_back + i * S * M * 2) for i in range(2)]
            if push1 else None,
            retbuf=None if push1 else region.tensor(off_back, (max(S * k, 1), M), torch.bfloat16),
            peer_retbuf=None if push1 else region.ptr_table(off_back), flip=0,
            signal=region.tensor(off_sig, (64,), torch.int32),
            signal2=region.tensor(off_sig2, (64,), torch.int32),
            counts=region.tensor(off_cnt, (self.world * C * self.E,), torch.int32),
            peer_cnt=region.ptr_table(off_cnt),
            peer_recv=region.ptr_table(off_recv), peer_tok=region.ptr_table(off_tok),
            peer_prob=region.ptr_table(off_prob),
            peer_ret=region.ptr_table(off_ret) if C > 1 else None,
            peer_sig=region.ptr_table(off_sig), peer_sig2=region.ptr_table(off_sig2),
            slot_base=torch.empty(C * self.E, **i32), row_base=torch.empty(C * self.E, **i32),
            seg_start=torch.empty(C * G, **i32), seg_rows=torch.empty(C * G, **i32),
            seg_w=torch.arange(G, **i32), recv_rows=torch.empty(C, **i32),
            totals_c=torch.empty(C * self.E, **i32), kept_c=torch.empty(C * self.E, **i32),
            h=torch.empty((rmax, self.F), dtype=self.dtype, device=self.dev),
            err=torch.zeros(1, **i32),
        )
        if self.shared is not None:  # the source's shared MLP: one group of S token rows
            st.update(hs=torch.empty((max(S, 1), self.F), dtype=self.dtype, device=self.dev),
                      sh_rows=torch.tensor([S], **i32), sh_w=torch.zeros(1, **i32))
        dist.barrier(group=self.group)
        self._p2p[S] = st
        return st

    def _barrier(self, st: dict, channel: int = 0) -> None:
        """Flag barrier of every rank on the current stream; channel 1 is the comm
        stream's (its own signals and epoch, so the two streams never interleave)."""
        sig, psig, ep = ((st["signal"], st["peer_sig"], self._epoch_dev) if channel == 0 else
                         (st["signal2"], st["peer_sig2"], self._epoch2_dev))
        _lib.call("moe_ipc_barrier", psig.data_ptr(), sig.data_ptr(), self.world, self.rank,
                  ep.data_ptr(), st["err"].data_ptr(), _lib.stream_ptr())

    def check_errors(self) -> None:
        """Raise if a peer barrier timed out (call after synchronising)."""
        for st in (self._p2p or {}).values():
            if int(st["err"].item()):
                raise RuntimeError("expert-parallel peer barrier timed out")

    def _forward_p2p(self, x: torch.Tensor, out: torch.Tensor | None, timer):
        """Peer-memory forward: gate -> counts all-gather over peer memory -> device
        plan -> dispatch straight into the owners' receive buffers -> barrier ->
        owner GEMM1 / GEMM2 whose epilogue stores every row back to its source over
        NVLink -> barrier -> (k=2 / Residual-MoE) local combine. k=1 layers without
        a shared MLP are combined by the owner's epilogue into the source's output
        slot (alternating between two per batch size; returned when ``out`` is None,
        copied into ``out`` otherwise)."""
        if self.chunks > 1:
            return self._forward_p2p_chunked(x, out, timer)
        if x.device != self.dev:
            x = x.to(self.dev, non_blocking=True)
        x = x.to(self.dtype).contiguous()
        if x.dim() != 2 or x.shape[1] != self.M:
            raise ShapeError(f"batch width {tuple(x.shape)} does not match layer hidden {self.M}")
        S = x.shape[0]
        ws = self._workspace(S)
        st = self._p2p_state(S)
        E, M, F, k, cap = self.E, self.M, self.F, self.k, st["cap"]
        stream = _lib.stream_ptr()
        ph = _Phases(timer)
        ids, gp, lr, tc = ws["ids"], ws["gp"], ws["local_rank"], ws["tile_counts"]
        push1 = st["push1"]
        if push1:
            j = st["flip"]
            st["flip"] ^= 1
            slot, dest = st["oslot"][j], st["peer_oslot"][j]
        else:
            slot, dest = None, st["peer_retbuf"]
            out = torch.empty_like(x) if out is None else out
        ph("gate")
        if S:
            _lib.call("moe_gate_gemm_bf16", x.data_ptr(), self.wg.data_ptr(), S, M, E, k, None,
                      ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), stream)
        ph("scan")
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, 2 ** 62, None,
                  ws["tile_offsets"].data_ptr(), ws["totals"].data_ptr(), ws["kept"].data_ptr(),
                  stream)
        ph("counts_allgather")
        # per-expert counts to every rank over peer memory; the fused barrier also
        # orders this step after every rank's previous step (buffer reuse)
        _lib.call("moe_ipc_allgather_i32", ws["totals"].data_ptr(), E, st["peer_cnt"].data_ptr(),
                  self.world, self.rank, st["peer_sig"].data_ptr(), st["signal"].data_ptr(),
                  self._epoch_dev.data_ptr(), st["err"].data_ptr(), stream)
        ph("plan")
        # padded receive layout (local expert j at rows [j*cap, (j+1)*cap)): the owner's
        # GEMMs run with a uniform group stride, like the single-GPU expert buffers
        _lib.call("moe_ep_plan_padded", st["counts"].data_ptr(), self.world, self.rank, E, cap,
                  st["slot_base"].data_ptr(), st["row_base"].data_ptr(),
                  st["seg_start"].data_ptr(), st["seg_rows"].data_ptr(),
                  st["recv_rows"].data_ptr(), stream)
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, cap, st["slot_base"].data_ptr(),
                  ws["tile_offsets"].data_ptr(), ws["totals"].data_ptr(), ws["kept"].data_ptr(),
                  stream)
        ph("dispatch_p2p")
        if S:
            _lib.call("moe_dispatch_p2p", x.data_ptr(), S, M * 2, E, k, cap, ids.data_ptr(),
                      lr.data_ptr(), ws["tile_offsets"].data_ptr(), gp.data_ptr(),
                      st["slot_base"].data_ptr(), st["row_base"].data_ptr(), self.E_loc,
                      st["peer_recv"].data_ptr(), st["peer_tok"].data_ptr(),
                      st["peer_prob"].data_ptr(), ws["slots"].data_ptr(),
                      ws["row_index"].data_ptr(), _lib.ptr(slot), st["peer_src"].data_ptr(),
                      self.rank, stream)
        self._barrier(st)
        G = self.E_loc
        if cap:
            # padding rows are scratch: TMA-store epilogue; 256-column tiles (the
            # 256 x 512 GELU tiles measured less even across ranks: the return
            # barrier waited 0.13-0.36 ms for the slower one, 0.02-0.06 ms on 256)
            ph("gemm1")
            _lib.call("moe_grouped_gemm_bf16", st["recv"].data_ptr(), st["rmax"], M,
                      self.w1.data_ptr(), self.E_loc * F, F, self.b1.data_ptr(),
                      st["h"].data_ptr(), G, None, cap, st["seg_rows"].data_ptr(), 0, None, cap,
                      _lib.MOE_ACT_GELU | _lib.MOE_GEMM_PAD_SCRATCH | _lib.MOE_GEMM_TILE256,
                      stream)
            # GEMM2 + bias (+ combine and residual for k=1), every row stored straight
            # back to its source rank over NVLink
            ph("gemm2_push")
            _lib.call("moe_grouped_gemm_bf16_push", st["h"].data_ptr(), st["rmax"], F,
                      self.w2.data_ptr(), self.E_loc * M, M, self.b2.data_ptr(), G, None, cap,
                      st["seg_rows"].data_ptr(), None, cap, 1 if push1 else 0,
                      st["row_token"].data_ptr(), st["row_prob"].data_ptr(),
                      st["row_src"].data_ptr(), dest.data_ptr(), st["recv"].data_ptr(), stream)
        if self.shared is not None and S:
            ph("shared_mlp1")  # the source's shared MLP, first half (replicated weights)
            sh = self.shared
            _lib.call("moe_grouped_gemm_bf16", x.data_ptr(), S, M, sh.w1.data_ptr(), F, F,
                      sh.b1.data_ptr(), st["hs"].data_ptr(), 1, None, 0, None, S, None, S,
                      _lib.MOE_ACT_GELU | _lib.MOE_GEMM_PAD_SCRATCH, stream)
        ph("return_barrier")
        self._barrier(st)
        if push1:
            ph(None)
            if out is None:
                return slot
            out.copy_(slot)
            return out
        if S:
            if self.shared is not None:
                # out = (x + sum_j p_j y_j) + shared MLP(x): the shared GEMM2 epilogue
                # reads the returned expert rows (arch.py:389-391)
                ph("shared_mlp2_combine")
                sh = self.shared
                _lib.call("moe_residual_gemm_bf16", st["hs"].data_ptr(), S, None, 0, 0, F,
                          sh.w2.data_ptr(), M, M, sh.b2.data_ptr(), st["retbuf"].data_ptr(), 1,
                          S, st["sh_rows"].data_ptr(), st["sh_w"].data_ptr(), S, 0, 0,
                          ids.data_ptr(), None, gp.data_ptr(), k, cap, x.data_ptr(),
                          out.data_ptr(), S, ws["row_index"].data_ptr(), stream)
            else:
                ph("combine")
                _lib.call("moe_combine", st["retbuf"].data_ptr(), _lib.MOE_BF16, S, M, E, k, cap,
                          ids.data_ptr(), ws["slots"].data_ptr(), ws["row_index"].data_ptr(),
                          gp.data_ptr(), _lib.MOE_F32, x.data_ptr(), None, out.data_ptr(), 1,
                          stream)
        ph(None)
        return out

    def _forward_p2p_chunked(self, x: torch.Tensor, out: torch.Tensor | None, timer):
        """p2p forward with every rank's tokens in C chunks, pipelined over two
        streams: the comm stream dispatches chunk c+1 and pulls chunk c-1's
        combined rows while the main stream runs chunk c's GEMMs on the SMs the
        launch limits leave free. Per-row results are the unchunked ones (same
        kernels on the same rows), so outputs stay bit-identical."""
        if x.device != self.dev:
            x = x.to(self.dev, non_blocking=True)
        x = x.to(self.dtype).contiguous()
        if x.dim() != 2 or x.shape[1] != self.M:
            raise ShapeError(f"batch width {tuple(x.shape)} does not match layer hidden {self.M}")
        S, C, RT = x.shape[0], self.chunks, _lib.ROUTE_TILE
        if S % (C * RT):
            raise ValueError(f"{C} chunks need tokens per rank in multiples of {C * RT}")
        ws = self._workspace(S)
        st = self._p2p_state(S)
        E, M, F, k, cap = self.E, self.M, self.F, self.k, st["cap"]
        Sc, Tc, G = S // C, S // C // RT, self.E_loc
        main = torch.cuda.current_stream(self.dev)
        if getattr(self, "_comm", None) is None:
            # GEMMs on a high-priority stream: when a chunk's GEMM and a copy kernel
            # become ready together, the block scheduler places the GEMM's CTAs first
            # and the copy kernel's (capped) blocks land on the SMs left free
            lo, hi = torch.cuda.Stream.priority_range()
            self._comm = torch.cuda.Stream(device=self.dev, priority=lo)
            self._gemm = torch.cuda.Stream(device=self.dev, priority=hi)
            self._nsm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        comm, gstream = self._comm, self._gemm
        ms = _lib.stream_ptr()
        ids, gp, lr, tc = ws["ids"], ws["gp"], ws["local_rank"], ws["tile_counts"]
        tof, slots, rix = ws["tile_offsets"], ws["slots"], ws["row_index"]
        out = torch.empty_like(x) if out is None else out
        rb = M * x.element_size()
        if S:
            _lib.call("moe_gate_gemm_bf16", x.data_ptr(), self.wg.data_ptr(), S, M, E, k, None,
                      ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), ms)
        tot, kep = st["totals_c"], st["kept_c"]
        for c in range(C):  # per-chunk expert counts
            _lib.call("moe_plan_scan", tc[c * Tc:].data_ptr(), Sc, E, 2 ** 62, None,
                      tof[c * Tc:].data_ptr(), tot[c * E:].data_ptr(), kep[c * E:].data_ptr(), ms)
        _lib.call("moe_ipc_allgather_i32", tot.data_ptr(), C * E, st["peer_cnt"].data_ptr(),
                  self.world, self.rank, st["peer_sig"].data_ptr(), st["signal"].data_ptr(),
                  self._epoch_dev.data_ptr(), st["err"].data_ptr(), ms)
        _lib.call("moe_ep_plan_chunked", st["counts"].data_ptr(), self.world, self.rank, E, C, cap,
                  st["slot_base"].data_ptr(), st["row_base"].data_ptr(), st["seg_start"].data_ptr(),
                  st["seg_rows"].data_ptr(), st["recv_rows"].data_ptr(), ms)
        for c in range(C):  # global slots of each chunk
            _lib.call("moe_plan_scan", tc[c * Tc:].data_ptr(), Sc, E, cap,
                      st["slot_base"][c * E:].data_ptr(), tof[c * Tc:].data_ptr(),
                      tot[c * E:].data_ptr(), kep[c * E:].data_ptr(), ms)
        R = self.comm_sms

        def dispatch(c, limited):
            _lib.call("moe_set_launch_limits", 0, R * 8 if limited else 0)
            _lib.call("moe_dispatch_p2p", x[c * Sc:].data_ptr(), Sc, rb, E, k, cap,
                      ids[c * Sc:].data_ptr(), lr[c * Sc:].data_ptr(), tof[c * Tc:].data_ptr(),
                      gp[c * Sc:].data_ptr(), st["slot_base"][c * E:].data_ptr(),
                      st["row_base"][c * E:].data_ptr(), G, st["peer_recv"].data_ptr(),
                      st["peer_tok"].data_ptr(), st["peer_prob"].data_ptr(),
                      slots[c * Sc:].data_ptr(), rix[c * Sc:].data_ptr(),
                      out[c * Sc:].data_ptr(), None, 0, _lib.stream_ptr())
            _lib.call("moe_set_launch_limits", 0, 0)
            self._barrier(st, channel=1)

        def pull(c, limited):
            _lib.call("moe_set_launch_limits", 0, R * 8 if limited else 0)
            _lib.call("moe_pull_rows_p2p", Sc, rb, E, k, ids[c * Sc:].data_ptr(),
                      rix[c * Sc:].data_ptr(), G, st["peer_ret"].data_ptr(),
                      out[c * Sc:].data_ptr(), _lib.stream_ptr())
            _lib.call("moe_set_launch_limits", 0, 0)

        fork = torch.cuda.Event()
        fork.record(main)
        comm.wait_event(fork)
        gstream.wait_event(fork)
        ev_d = [torch.cuda.Event() for _ in range(C)]
        ev_g = [torch.cuda.Event() for _ in range(C)]
        with torch.cuda.stream(comm):
            dispatch(0, False)
            ev_d[0].record(comm)
        try:
            self._chunk_loop(C, cap, st, dispatch, pull, ev_d, ev_g, comm, gstream, main)
        finally:
            torch.cuda.set_stream(main)
        for s_ in (comm, gstream):
            join = torch.cuda.Event()
            join.record(s_)
            main.wait_event(join)
        return out

    def _chunk_loop(self, C, cap, st, dispatch, pull, ev_d, ev_g, comm, gstream, main):
        M, F, G, R = self.M, self.F, self.E_loc, self.comm_sms
        for c in range(C):
            gstream.wait_event(ev_d[c])
            torch.cuda.set_stream(gstream)
            ms = _lib.stream_ptr()
            if cap:
                _lib.call("moe_set_launch_limits", self._nsm - R, 0)
                _lib.call("moe_grouped_gemm_bf16", st["recv"].data_ptr(), st["rmax"], M,
                          self.w1.data_ptr(), G * F, F, self.b1.data_ptr(), st["h"].data_ptr(), G,
                          st["seg_start"][c * G:].data_ptr(), 0, st["seg_rows"][c * G:].data_ptr(),
                          0, st["seg_w"].data_ptr(), cap, _lib.MOE_ACT_GELU, ms)
                _lib.call("moe_grouped_gemm_bf16_combine_rows", st["h"].data_ptr(), st["rmax"], F,
                          self.w2.data_ptr(), G * M, M, self.b2.data_ptr(), G,
                          st["seg_start"][c * G:].data_ptr(), st["seg_rows"][c * G:].data_ptr(),
                          st["seg_w"].data_ptr(), cap, st["row_token"].data_ptr(),
                          st["row_prob"].data_ptr(), st["recv"].data_ptr(), st["ret"].data_ptr(),
                          ms)
                _lib.call("moe_set_launch_limits", 0, 0)
            self._barrier(st, channel=0)
            ev_g[c].record(gstream)
            torch.cuda.set_stream(main)
            with torch.cuda.stream(comm):
                if c + 1 < C:
                    dispatch(c + 1, True)
                    ev_d[c + 1].record(comm)
                comm.wait_event(ev_g[c])
                pull(c, c + 1 < C)

    def plan(self, S: int):
        """(ids, gate_probs, global slots, plan) of the last forward; for the p2p
        transport the plan is summarised as (cap, expert_load) from device tables."""
        ws = self._ws[S]
        if self.transport == "p2p":
            from types import SimpleNamespace

            self.check_errors()
            st = self._p2p[S]
            load = st["seg_rows"].cpu().numpy()
            load = load.reshape(self.chunks, self.E_loc).sum(axis=0)
            return ws["ids"], ws["gp"], ws["slots"], SimpleNamespace(cap=st["cap"],
                                                                     expert_load=load)
        return ws["ids"], ws["gp"], ws["slots"], self.last_plan


class SlicedEPMoeLayer(EPMoeLayer):
    """MoE layer over tensor-sliced groups with expert slicing (bf16, NCCL).

    Ranks form Q = world / L groups of L consecutive ranks (tensor_slice L,
    planner.py:160-174: groups never span nodes); the members of a group hold
    the same token shard. Group q owns experts [q*E/Q, (q+1)*E/Q) and member t
    of the group holds d_ff slice [t*F/L, (t+1)*F/L) of each of them: W1
    columns, b1 and W2 rows of the slice (b2 on member 0), so
      y = sum_t gelu(x W1_t + b1_t) W2_t + b2      (expert slicing, planner.py:207-222).
    Forward: gate + global-capacity plan over the Q groups (the replicas must
    agree - ReplicaMismatchError otherwise, commsim.py:404-411), coordinated
    dispatch (commsim.py:373-464), per-slice GEMMs, all-reduce of the partial
    outputs inside the group, coordinated return, combine. Routing and slots
    equal the single-GPU layer on the concatenated group shards bit-exactly;
    outputs differ from it only by the bf16 rounding of the slice partials."""

    def __init__(self, spec: LayerSpec, gate_w, group_experts, shared=None, group=None,
                 tensor_slice: int = 2, dtype=torch.bfloat16, device=None) -> None:
        if spec.kind != "moe":
            raise ShapeError("SlicedEPMoeLayer needs a moe LayerSpec")
        if dtype != torch.bfloat16:
            raise TypeError("the expert-parallel path is bf16 (tcgen05)")
        if spec.residual:
            raise ValueError("the sliced layer covers layers without the Residual-MoE shared MLP")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        L = int(tensor_slice)
        if L < 1 or self.world % L:
            raise ValueError(f"tensor_slice {tensor_slice} must divide world {self.world}")
        self.L, self.Q = L, self.world // L
        self.q, self.t = divmod(self.rank, L)
        E, M = spec.experts, spec.hidden
        F = FFN_MULT * M
        if E % self.Q:
            raise ValueError(f"{E} experts do not divide over {self.Q} groups (planner.py:202-206)")
        if F % L or (F // L) % 8:
            raise ValueError(f"d_ff {F} does not slice into {L} multiples of 8")
        dev = _lib.require_device(None) if device is None else torch.device(device)
        self.spec, self.dev, self.dtype = spec, dev, dtype
        self.E, self.M, self.F, self.k = E, M, F, spec.gating.k
        self.E_loc = E // self.Q
        self.Fs = Fs = F // L
        if len(group_experts) != self.E_loc:
            raise ShapeError(f"{len(group_experts)} group experts, expected {self.E_loc}")
        gw = _t(gate_w, dev, torch.float32)
        self.epad = max(32, 1 << (E - 1).bit_length())
        self.wg = torch.zeros((self.epad, M), dtype=torch.bfloat16, device=dev)
        self.wg[:E] = gw.t().to(torch.bfloat16)
        lo, hi = self.t * Fs, (self.t + 1) * Fs
        self.w1 = torch.empty((self.E_loc * Fs, M), dtype=torch.bfloat16, device=dev)
        self.w2 = torch.empty((self.E_loc * M, Fs), dtype=torch.bfloat16, device=dev)
        self.b1 = torch.empty((self.E_loc, Fs), dtype=torch.float32, device=dev)
        self.b2 = torch.zeros((self.E_loc, M), dtype=torch.float32, device=dev)
        for i, p in enumerate(group_experts):
            self.w1[i * Fs:(i + 1) * Fs] = _t(p.w1, dev, torch.bfloat16)[:, lo:hi].t()
            self.w2[i * M:(i + 1) * M] = _t(p.w2, dev, torch.bfloat16)[lo:hi].t()
            self.b1[i] = _t(p.b1, dev, torch.float32).reshape(F)[lo:hi]
            if self.t == 0:  # the output bias once per group
                self.b2[i] = _t(p.b2, dev, torch.float32).reshape(M)
        self.shared = None
        self.transport, self.schedule = "nccl", "coordinated"
        self.exchanger = Exchanger(group, "coordinated", tensor_slice=L)
        self._ws: dict = {}
        self._p2p = None
        self._pipe = None
        self.last_plan: ExchangePlan | None = None

    @classmethod
    def from_params(cls, spec: LayerSpec, params: MoeLayerParams, group=None, tensor_slice: int = 2,
                    **kw):
        """This group's expert block out of full (replicated) parameters."""
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        Q = world // tensor_slice
        e_loc = spec.experts // Q
        q = rank // tensor_slice
        local = params.experts[q * e_loc:(q + 1) * e_loc]
        return cls(spec, params.gate_w, local, params.shared, group=group,
                   tensor_slice=tensor_slice, **kw)

    def graphed(self, S: int):
        raise NotImplementedError("the sliced layer syncs counts on the host (NCCL splits)")

    def kept_assignments(self, S: int) -> int:
        return int(self.last_plan.kept[self.q].sum()) if self.last_plan is not None else 0

    def _forward_dev(self, x: torch.Tensor, out: torch.Tensor | None = None, timer=None):
        if x.device != self.dev:
            x = x.to(self.dev, non_blocking=True)
        x = x.to(self.dtype).contiguous()
        if x.dim() != 2 or x.shape[1] != self.M:
            raise ShapeError(f"batch width {tuple(x.shape)} does not match layer hidden {self.M}")
        S = x.shape[0]
        out = torch.empty_like(x) if out is None else out
        ws = self._workspace(S)
        E, M, Fs, k, L, Q = self.E, self.M, self.Fs, self.k, self.L, self.Q
        st = _lib.stream_ptr()
        ph = _Phases(timer)
        ids, gp, lr, tc = ws["ids"], ws["gp"], ws["local_rank"], ws["tile_counts"]
        ph("gate")
        if S:
            _lib.call("moe_gate_gemm_bf16", x.data_ptr(), self.wg.data_ptr(), S, M, E, k, None,
                      ids.data_ptr(), gp.data_ptr(), lr.data_ptr(), tc.data_ptr(), st)
        ph("scan")
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, 2 ** 62, None,
                  ws["tile_offsets"].data_ptr(), ws["totals"].data_ptr(), ws["kept"].data_ptr(),
                  st)
        ph("counts_allgather")
        counts = gather_counts(ws["counts"], ws["totals"], self.group).cpu().numpy()
        counts = counts.reshape(Q, L, E)
        if not (counts == counts[:, :1]).all():
            raise ReplicaMismatchError("members of a tensor group routed different token shards")
        gcounts = counts[:, 0]
        s_total = int(gcounts.sum()) // k
        cap = self.spec.gating.capacity(s_total)
        plan = make_exchange_plan(gcounts, cap, self.q, E)  # groups play the ranks
        self.last_plan = plan
        ph("scan")
        G = Q * self.E_loc
        tables = np.concatenate([plan.base[self.q], plan.send_row_base, plan.seg_row_start,
                                 plan.seg_rows, plan.seg_weight]).astype(np.int32)
        tab = torch.from_numpy(tables).to(self.dev, non_blocking=True)
        base_d, row_base_d = tab[:E], tab[E:2 * E]
        seg_start_d, seg_rows_d, seg_w_d = tab[2 * E:2 * E + G], tab[2 * E + G:2 * E + 2 * G], \
            tab[2 * E + 2 * G:2 * E + 3 * G]
        _lib.call("moe_plan_scan", tc.data_ptr(), S, E, cap, base_d.data_ptr(),
                  ws["tile_offsets"].data_ptr(), ws["totals"].data_ptr(), ws["kept"].data_ptr(),
                  st)
        ph("dispatch")
        if S:
            _lib.call("moe_dispatch_ep", x.data_ptr(), S, M * 2, E, k, cap, ids.data_ptr(),
                      lr.data_ptr(), ws["tile_offsets"].data_ptr(), base_d.data_ptr(),
                      row_base_d.data_ptr(), ws["slots"].data_ptr(), ws["row_index"].data_ptr(),
                      ws["send"].data_ptr(), st)
        ph("coordinated_dispatch")
        n_recv = plan.n_recv
        if ws.get("recv_rows", -1) < n_recv:
            rows = max(n_recv, 1)
            ws["recv"] = torch.empty((rows, M), dtype=self.dtype, device=self.dev)
            ws["h"] = torch.empty((rows, Fs), dtype=self.dtype, device=self.dev)
            ws["y"] = torch.empty((rows, M), dtype=self.dtype, device=self.dev)
            ws["recv_rows"] = rows
        Cg = rank_counts(plan)
        recv = self.exchanger.coordinated(ws["recv"], ws["send"], Cg)
        max_rows = int(plan.seg_rows.max()) if plan.seg_rows.size else 0
        y = ws["y"][:n_recv]
        if n_recv and max_rows:
            ph("gemm1_slice")
            _lib.call("moe_grouped_gemm_bf16", recv.data_ptr(), n_recv, M, self.w1.data_ptr(),
                      self.E_loc * Fs, Fs, self.b1.data_ptr(), ws["h"].data_ptr(), G,
                      seg_start_d.data_ptr(), 0, seg_rows_d.data_ptr(), 0, seg_w_d.data_ptr(),
                      max_rows, _lib.MOE_ACT_GELU, st)
            ph("gemm2_slice")
            _lib.call("moe_grouped_gemm_bf16", ws["h"].data_ptr(), n_recv, Fs, self.w2.data_ptr(),
                      self.E_loc * M, M, self.b2.data_ptr(), y.data_ptr(), G,
                      seg_start_d.data_ptr(), 0, seg_rows_d.data_ptr(), 0, seg_w_d.data_ptr(),
                      max_rows, _lib.MOE_ACT_NONE, st)
            if L > 1:
                ph("slice_allreduce")
                all_reduce_sum(y, group=self.exchanger.slice_group)
        ph("coordinated_return")
        self.exchanger.coordinated(ws["ret"], ws["y"], Cg.T)
        ph("combine")
        if S:
            _lib.call("moe_combine", ws["ret"].data_ptr(), _lib.MOE_BF16, S, M, E, k, cap,
                      ids.data_ptr(), ws["slots"].data_ptr(), ws["row_index"].data_ptr(),
                      gp.data_ptr(), _lib.MOE_F32, x.data_ptr(), None, out.data_ptr(), 1, st)
        ph(None)
        return out
