"""Per-call device time of FastComm.alltoallv with and without PDL on the
call chain, small (latency) and config-2 (256 MiB Zipf 1.2) traffic.
torchrun --nproc-per-node N tools/pdl_ab.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2505_09764_b200 import Topology, workloads
from paper_2505_09764_b200.executor import FastComm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n, m = 2, world // 2
for name, D in (("hotspot 512 B mean", workloads.gen_hotspot(3, Topology(n, m), 512, hot=0, factor=8).sizes),
                ("config2 256 MiB", workloads.zipf_sizes(0, world, 1.2, 268_435_456))):
    cap = int(max(D.sum(0).max(), D.sum(1).max())) + 4096
    comm = FastComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (4 << 20))
    send = torch.zeros(int(D[rank].sum()) + 16, dtype=torch.uint8, device="cuda")
    row = torch.from_numpy(D[rank].copy()).cuda()
    for pdl in (False, True, False, True):
        comm.set_pdl(pdl)
        for _ in range(20):
            comm.alltoallv(send, row)
        torch.cuda.synchronize(); dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 200 if cap < (1 << 24) else 30
        a.record()
        for _ in range(K):
            comm.alltoallv(send, row)
        b.record(); torch.cuda.synchronize()
        comm.check()
        t = torch.tensor([a.elapsed_time(b) / K * 1e3], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(f"{name:22s} pdl={pdl!s:5s}: {t.item():8.1f} us per call", flush=True)
    comm.close()
dist.destroy_process_group()
