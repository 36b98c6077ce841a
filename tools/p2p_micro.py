"""NVLink envelope of the exec kernel: FastComm on synthetic patterns.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/p2p_micro.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2505_09764_b200 import Topology
from paper_2505_09764_b200.executor import FastComm

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
SZ = 256 << 20
blocks = int(os.environ.get("BLOCKS", "148"))
chunk = int(os.environ.get("CHUNK", str(1 << 20)))
pats = {}
G = world
D = np.zeros((G, G), np.int64); D[0, 1] = SZ; pats["0->1"] = D
D = np.zeros((G, G), np.int64); D[0, 1] = SZ; D[1, 0] = SZ; pats["0<->1"] = D
if G >= 4:
    D = np.zeros((G, G), np.int64); D[0, 1:] = SZ // (G - 1); pats["0->all"] = D
    D = np.zeros((G, G), np.int64); D[1:, 0] = SZ // (G - 1); pats["all->0"] = D
    D = np.full((G, G), SZ // (G - 1), np.int64); np.fill_diagonal(D, 0); pats["uniform"] = D
    D = np.zeros((G, G), np.int64)
    for g in range(G): D[g, (g + 1) % G] = SZ
    pats["ring"] = D
comm = FastComm(Topology(G, 1), recv_bytes=SZ + 4096, staging_bytes=1 << 20, blocks=blocks,
                chunk_bytes=chunk)
send = torch.randint(0, 256, (SZ + 16,), dtype=torch.uint8, device="cuda")
for name, D in pats.items():
    row = torch.from_numpy(D[rank].copy()).cuda()
    for _ in range(3):
        comm.alltoallv(send, row)
    torch.cuda.synchronize(); dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for a, b in ev:
        comm.alltoallv(send, row, exec_events=(a, b))
    torch.cuda.synchronize(); comm.check()
    ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / len(ev)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    bn = max(D.sum(0).max(), D.sum(1).max())
    out = torch.empty(int(D[:, rank].sum()) + 16, dtype=torch.uint8, device="cuda")
    ins, outs = D[rank].tolist(), D[:, rank].tolist()
    sv = send[: int(D[rank].sum())]
    ov = out[: int(D[:, rank].sum())]
    for _ in range(3):
        dist.all_to_all_single(ov, sv, outs, ins)
    torch.cuda.synchronize(); dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        dist.all_to_all_single(ov, sv, outs, ins)
    b.record(); torch.cuda.synchronize()
    nm = torch.tensor([a.elapsed_time(b) / 10], device="cuda")
    dist.all_reduce(nm, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"{name:8s} bottleneck {bn/2**20:.0f} MiB  exec {ms.item()*1e3:.1f} us  "
              f"{bn/(ms.item()*1e-3)/1e9:.1f} GB/s per bottleneck direction; "
              f"NCCL {nm.item()*1e3:.1f} us {bn/(nm.item()*1e-3)/1e9:.1f} GB/s", flush=True)
comm.close()
dist.destroy_process_group()
