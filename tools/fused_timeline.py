"""Where a small FastComm call's time goes, fused single-launch path vs the
multi-launch chain: exec-kernel %globaltimer stamps (ns since kernel start).
torchrun --nproc-per-node 2 tools/fused_timeline.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2505_09764_b200 import Topology, workloads
from paper_2505_09764_b200.executor import FastComm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n, m = 2, world // 2
D = workloads.gen_hotspot(3, Topology(n, m), 512, hot=0, factor=8).sizes
comm = FastComm(Topology(n, m), recv_bytes=1 << 20, staging_bytes=1 << 20)
send = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
row = torch.from_numpy(D[rank].copy()).cuda()
for fused in (True, False):
    comm.set_fused(fused)
    comm.use_graph = True
    acc = np.zeros(16)
    for it in range(60):
        comm.alltoallv(send, row, record_timeline=True)
        torch.cuda.synchronize()
        if it >= 20:
            t = comm.timeline.cpu().numpy().astype(np.int64)
            base = t[0]
            acc += np.array([t[i] - base if t[i] else 0 for i in range(16)])
    comm.check()
    a = acc / 40 / 1e3
    # events-based per-call time
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record()
    for _ in range(100):
        comm.alltoallv(send, row)
    ev[1].record(); torch.cuda.synchronize()
    if rank == 0:
        print(f"fused={fused}: per call {ev[0].elapsed_time(ev[1]) / 100 * 1e3:.1f} us; stamps us since "
              f"kernel start: prologue start {a[5]:.1f} gathered {a[6]:.1f} balanced {a[7]:.1f} "
              f"decomposed {a[12]:.1f} barrier {a[1]:.1f} recv_done {a[4]:.1f}", flush=True)
comm.close(); dist.destroy_process_group()
