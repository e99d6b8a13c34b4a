"""Host <-> device streaming for layers called with host tensors.

A layer called with a (pinned) host batch copies it in on an H2D stream into
one of two device staging buffers, runs the forward on the caller's stream,
and copies the result out on a D2H stream from one of two device output
buffers. With two slots, step i+1's upload and step i-1's download overlap
step i's kernels (the copy engines of each direction are separate), so a
stream of batches runs at max(H2D, compute, D2H) per batch instead of their
sum. Every call is asynchronous; results are valid once the caller syncs
(``torch.cuda.synchronize()`` or ``HostPipeline.wait()``).
"""

from __future__ import annotations

import torch


class HostPipeline:
    def __init__(self, fn, width: int, dtype: torch.dtype, device) -> None:
        self.fn, self.width, self.dtype, self.device = fn, width, dtype, device
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.rows = -1
        self.slot = 0
        self.x_dev = [None, None]
        self.y_dev = [None, None]
        self.ev_in = [torch.cuda.Event() for _ in range(2)]       # upload into slot done
        self.ev_used = [torch.cuda.Event() for _ in range(2)]     # compute reading slot done
        self.ev_out = [torch.cuda.Event() for _ in range(2)]      # download from slot done
        self.started = [False, False]

    def _alloc(self, rows: int) -> None:
        if rows == self.rows:
            return
        # the old slots may still be read by an in-flight copy on either copy stream
        # (the caching allocator would hand them out again to this stream at once)
        torch.cuda.current_stream(self.device).synchronize()
        self.h2d.synchronize()
        self.d2h.synchronize()
        self.x_dev = [torch.empty((rows, self.width), dtype=self.dtype, device=self.device)
                      for _ in range(2)]
        self.y_dev = [torch.empty((rows, self.width), dtype=self.dtype, device=self.device)
                      for _ in range(2)]
        self.rows = rows
        self.started = [False, False]

    def __call__(self, x_host: torch.Tensor, out_host: torch.Tensor | None = None, **kw):
        rows = x_host.shape[0]
        self._alloc(rows)
        j = self.slot
        self.slot ^= 1
        cur = torch.cuda.current_stream(self.device)
        if out_host is None:
            out_host = torch.empty((rows, self.width), dtype=self.dtype, pin_memory=True)
        # upload: the staging slot must no longer be read by the previous forward
        if self.started[j]:
            self.h2d.wait_event(self.ev_used[j])
        with torch.cuda.stream(self.h2d):
            self.x_dev[j].copy_(x_host, non_blocking=True)
            self.ev_in[j].record(self.h2d)
        # compute: needs the upload, and the output slot must be downloaded already
        cur.wait_event(self.ev_in[j])
        if self.started[j]:
            cur.wait_event(self.ev_out[j])
        # (a layer may return its own output buffer instead of y_dev[j], e.g. the
        # EP peer-memory output slots, which alternate in step with this pipeline)
        y = self.fn(self.x_dev[j], out=self.y_dev[j], **kw)
        self.ev_used[j].record(cur)
        # download
        self.d2h.wait_event(self.ev_used[j])
        with torch.cuda.stream(self.d2h):
            out_host.copy_(y, non_blocking=True)
            self.ev_out[j].record(self.d2h)
        self.started[j] = True
        return out_host

    def wait(self) -> None:
        """Make the caller's stream wait for every outstanding download."""
        cur = torch.cuda.current_stream(self.device)
        for j in range(2):
            if self.started[j]:
                cur.wait_event(self.ev_out[j])


class GraphedForward:
    """A layer forward for one fixed batch shape, captured into a CUDA graph.

    Every kernel of the forward is stream-ordered with no host sync (the EP
    peer-memory barrier keeps its epoch on the device), so the whole layer
    replays as one graph launch: for decode-sized batches this removes the
    per-kernel launch and tensor-map encoding overheads. ``__call__`` copies
    the batch into the static input and returns the static output (valid until
    the next replay)."""

    def __init__(self, layer, rows: int, width: int, dtype: torch.dtype, device,
                 warmup: int = 2) -> None:
        self.x = torch.zeros((rows, width), dtype=dtype, device=device)
        self.out = torch.empty_like(self.x)
        side = torch.cuda.Stream(device=device)
        side.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.stream(side):  # allocate workspaces / one-time setup outside capture
            for _ in range(warmup):
                layer(self.x, out=self.out)
        torch.cuda.current_stream(device).wait_stream(side)
        torch.cuda.synchronize(device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.y = layer(self.x, out=self.out)
        # the captured kernels write into the layer's per-size workspaces: keep them
        # alive even if the layer later evicts them for other batch sizes (a replay
        # would otherwise write into memory the allocator has handed out again)
        self._keep = [d.get(rows) for d in (getattr(layer, "_ws", None),
                                            getattr(layer, "_p2p", None)) if d]

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        self.x.copy_(x, non_blocking=True)
        self.graph.replay()
        return self.y
