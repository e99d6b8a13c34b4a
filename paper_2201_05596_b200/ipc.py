"""Peer-memory regions shared by the ranks of a process group (one GPU each).

Each rank cudaMallocs a region through libmoe_b200 (``moe_ipc_malloc``),
all-gathers the 64-byte cudaIpc handles over the group (NCCL; gloo when several
ranks share one GPU, which cudaIpc also supports), and opens the
peers' handles, so every rank holds device pointers to every rank's region:
NVLink loads/stores from kernels then go straight to the owner's HBM.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter, to view raw device memory as torch."""

    def __init__(self, ptr: int, shape, typestr: str) -> None:
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


_TYPESTR = {torch.int32: "<i4", torch.float32: "<f4", torch.int16: "<i2", torch.uint8: "|u1",
            torch.int64: "<i8"}


def view(ptr: int, shape, dtype: torch.dtype, device) -> torch.Tensor:
    """A torch tensor aliasing device memory at ``ptr`` (no ownership)."""
    if dtype == torch.bfloat16:
        return view(ptr, shape, torch.int16, device).view(torch.bfloat16)
    t = torch.as_tensor(_CudaArray(ptr, shape, _TYPESTR[dtype]), device=device)
    assert t.data_ptr() == ptr
    return t


class IpcRegion:
    """``nbytes`` of device memory on every rank, each mapped into every rank."""

    def __init__(self, nbytes: int, group=None, device=None) -> None:
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.nbytes = int(nbytes)
        lib = _lib.load()
        p = ctypes.c_void_p()
        _lib.check(lib.moe_ipc_malloc(self.nbytes, ctypes.addressof(p)), "moe_ipc_malloc")
        self.local = p.value
        h = (ctypes.c_uint8 * 64)()
        _lib.check(lib.moe_ipc_get_handle(self.local, ctypes.addressof(h)), "moe_ipc_get_handle")
        from .exchange import all_gather_flat

        mine = torch.tensor(np.frombuffer(bytes(h), dtype=np.uint8), device=self.device)
        allh = torch.empty(self.world * 64, dtype=torch.uint8, device=self.device)
        all_gather_flat(allh, mine, group=group)
        allh = allh.cpu().numpy().reshape(self.world, 64)
        self.ptrs = []
        for r in range(self.world):
            if r == self.rank:
                self.ptrs.append(self.local)
                continue
            hb = (ctypes.c_uint8 * 64)(*allh[r].tolist())
            q = ctypes.c_void_p()
            _lib.check(lib.moe_ipc_open_handle(ctypes.addressof(hb), ctypes.addressof(q)),
                       "moe_ipc_open_handle")
            self.ptrs.append(q.value)
        self._closed = False

    def ptr_table(self, offset: int) -> torch.Tensor:
        """Device int64 array of every rank's region base + offset."""
        return torch.tensor([p + offset for p in self.ptrs], dtype=torch.int64, device=self.device)

    def tensor(self, offset: int, shape, dtype: torch.dtype) -> torch.Tensor:
        return view(self.local + offset, shape, dtype, self.device)

    def close(self) -> None:
        if self._closed:
            return
        lib = _lib.load()
        torch.cuda.synchronize(self.device)
        for r, p in enumerate(self.ptrs):
            if r != self.rank:
                lib.moe_ipc_close_handle(p)
        lib.moe_ipc_free(self.local)
        self._closed = True

    def __del__(self) -> None:  # pragma: no cover - best effort at interpreter exit
        try:
            self.close()
        except Exception:
            pass
