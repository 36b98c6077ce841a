"""Push (peer stores) vs pull (peer loads) bandwidth of the executor's copy loop.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_rw.py
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2505_09764_b200 import Topology, _lib
from paper_2505_09764_b200.executor import FastComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
SZ = 256 << 20
comm = FastComm(Topology(world, 1), recv_bytes=2 * SZ, staging_bytes=2 * SZ, blocks=8)
lib = _lib.load()
me = lib.fast_comm_peer_ptr(comm._ptr, rank)
peer = lib.fast_comm_peer_ptr(comm._ptr, (rank + 1) % world)
recv_off = lib.fast_comm_recv_ptr(comm._ptr) - me
local = torch.randint(0, 256, (SZ,), dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()

def run(name, dst, src, active, blocks, chunk, nc):
    for _ in range(3):
        if active: lib.fast_debug_copy(dst, src, SZ, blocks, chunk, nc, ctypes.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize(); dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        if active: lib.fast_debug_copy(dst, src, SZ, blocks, chunk, nc, ctypes.c_void_p(stream.cuda_stream))
    b.record(); torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / 10 if active else 0.0], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"{name:28s} blocks={blocks:3d} chunk={chunk>>10:5d}K  {SZ/(ms.item()*1e-3)/1e9:7.1f} GB/s", flush=True)

for blocks in (132, 148, 296):
    for chunk in (1 << 20, 4 << 20):
        run("push 0->1 (peer store)", ctypes.c_void_p(peer + recv_off), ctypes.c_void_p(local.data_ptr()), rank == 0, blocks, chunk, 1)
        run("pull 1<-0 (peer load)", ctypes.c_void_p(me + recv_off), ctypes.c_void_p(peer), rank == 1 - 0 and rank == 1, blocks, chunk, 0)
        run("push both directions", ctypes.c_void_p(peer + recv_off), ctypes.c_void_p(local.data_ptr()), True, blocks, chunk, 1)
        run("pull both directions", ctypes.c_void_p(me + recv_off), ctypes.c_void_p(peer), True, blocks, chunk, 0)
comm.close()
dist.destroy_process_group()
