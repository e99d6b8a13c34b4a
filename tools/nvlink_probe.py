"""NVLink push/pull bandwidth probe (torchrun, >= 2 ranks): every rank moves
256 MB to / from its ring neighbour at the same time, (a) with the copy engine
(cudaMemcpyAsync into the peer's IPC-mapped buffer), (b) with SM remote stores
(moe_gather_rows writing the peer buffer, 16 B per lane), (c) with SM remote
loads (moe_gather_rows reading the peer buffer)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2201_05596_b200 import _lib  # noqa: E402
from paper_2201_05596_b200.ipc import IpcRegion, view  # noqa: E402

dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", torch.cuda.current_device())
NB = 256 << 20
ROW = 4096
rows = NB // ROW
reg = IpcRegion(NB, device=dev)
peer = (rank + 1) % world
peer_buf = view(reg.ptrs[peer], (rows, ROW // 2), torch.bfloat16, dev)
mine = reg.tensor(0, (rows, ROW // 2), torch.bfloat16)
src = torch.randn(rows, ROW // 2, device=dev).to(torch.bfloat16)
dst = torch.empty_like(src)
idx = torch.arange(rows, dtype=torch.int32, device=dev)
st = _lib.stream_ptr()


def ce():
    peer_buf.copy_(src)


def sm_push():
    _lib.call("moe_gather_rows", src.data_ptr(), ROW, idx.data_ptr(), rows, peer_buf.data_ptr(), st)


def sm_pull():
    _lib.call("moe_gather_rows", peer_buf.data_ptr(), ROW, idx.data_ptr(), rows, dst.data_ptr(), st)


def local():
    _lib.call("moe_gather_rows", src.data_ptr(), ROW, idx.data_ptr(), rows, dst.data_ptr(), st)


res = {}
for name, fn in (("copy_engine_push", ce), ("sm_push", sm_push), ("sm_pull", sm_pull), ("local_copy", local)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / 10], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    res[name] = {"ms": round(float(ms), 4), "GB_s_per_gpu": round(NB / float(ms) / 1e6, 1)}
    dist.barrier()
if rank == 0:
    print(json.dumps({"world": world, "bytes": NB, **res}))
torch.cuda.synchronize()
dist.barrier()
reg.close()
dist.destroy_process_group()
