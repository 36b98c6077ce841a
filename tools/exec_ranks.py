"""Per-rank exec timeline (globaltimer) and wire bytes for a config-2 call.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/exec_ranks.py [topo]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2505_09764_b200 import Topology, workloads
from paper_2505_09764_b200.executor import FastComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n, m = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else f"2x{world//2}").split("x"))
D = workloads.zipf_sizes(0, world, 1.2, 268_435_456)
cap = int(max(D.sum(0).max(), D.sum(1).max())) + 4096
comm = FastComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (4 << 20))
send = torch.randint(0, 256, (int(D[rank].sum()) + 16,), dtype=torch.uint8, device="cuda")
row = torch.from_numpy(D[rank].copy()).cuda()
for _ in range(5):
    comm.alltoallv(send, row, record_timeline=True)
torch.cuda.synchronize()
acc = np.zeros(3)
for _ in range(10):
    comm.alltoallv(send, row, record_timeline=True)
    torch.cuda.synchronize()
    t = comm.timeline.cpu().numpy().astype(np.float64)
    acc += [t[1] - t[0], t[3] - t[1], t[4] - t[1]]
acc /= 10
ops = comm.plan.host_ops()
eg = int(ops["len"][(ops["exec_rank"] == rank) & (ops["dst_rank"] != rank)].sum())
ing = int(ops["len"][(ops["dst_rank"] == rank) & (ops["exec_rank"] != rank)].sum())
by_phase = {p: int(ops["len"][(ops["exec_rank"] == rank) & (ops["phase"] == p)].sum()) for p in range(4)}
res = [None] * world
dist.all_gather_object(res, (rank, acc.tolist(), eg, ing, by_phase))
if rank == 0:
    print(f"topology {n}x{m}; direct bottleneck {max(D.sum(0).max(), D.sum(1).max())/1e6:.1f} MB")
    for r, a, eg, ing, bp in res:
        print(f"rank {r}: barrier {a[0]/1e3:6.1f} us  own-ops {a[1]/1e3:6.1f} us  recv-complete {a[2]/1e3:6.1f} us | "
              f"egress {eg/1e6:6.1f} MB ({eg/a[1]:.0f} GB/s over own-ops)  ingress {ing/1e6:6.1f} MB | phase bytes {bp}", flush=True)
comm.close(); dist.destroy_process_group()
