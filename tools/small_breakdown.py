"""Per-stage device time of one small FastComm alltoallv (config-4 style
hotspot, 512-byte cells), step by step with CUDA events between the stages:
gather | balance | decompose | sort | plan | exec.  Run with torchrun, N ranks.
Serialised stages (no PDL overlap), so the sum exceeds the chained call."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2505_09764_b200 import Topology, _lib, workloads  # noqa: E402
from paper_2505_09764_b200.executor import FastComm  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
topo = Topology(2, world // 2) if len(sys.argv) < 2 else Topology(*map(int, sys.argv[1].split("x")))
n, m = topo.n_servers, topo.gpus_per_server
D = workloads.gen_hotspot(3, topo, 512, hot=0, factor=8).sizes
comm = FastComm(topo, recv_bytes=1 << 20, staging_bytes=1 << 20)
send = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
row = torch.from_numpy(D[rank].copy()).cuda()
lib = _lib.load()
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
names = ["gather", "balance", "decompose", "sort", "plan", "exec"]
acc = np.zeros(len(names) + 1)
for _ in range(20):
    comm.alltoallv(send, row)
torch.cuda.synchronize()
dist.barrier()
for it in range(140):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    for x in ev:  # torch creates the CUDA event lazily, on its first record
        x.record(s)
    comm.epoch += 1
    e = comm.epoch
    ev[0].record(s)
    _lib.check_rc(lib.fast_gather_demand(comm._ptr, ctypes.c_void_p(row.data_ptr()), e, sh), "gather")
    ev[1].record(s)
    dptr = lib.fast_comm_demand_ptr(comm._ptr, e)
    kev = (ctypes.c_void_p * 4)(ev[1].cuda_event, ev[2].cuda_event, ev[3].cuda_event,
                                 ev[4].cuda_event)
    _lib.check_rc(lib.fast_synth_batch_ev(ctypes.c_void_p(dptr), 1, n, m,
                                          ctypes.byref(comm.sched.struct), sh, kev), "synth")
    ev[5].record(s)
    _lib.check_rc(lib.fast_plan_compile_ex(ctypes.c_void_p(dptr),
                                           ctypes.c_void_p(dptr + 8 * world * world), n, m,
                                           ctypes.byref(comm.sched.struct), comm.recv_bytes,
                                           comm.staging_bytes, comm.chunk,
                                           ctypes.byref(comm.plan.struct), 0, sh), "plan")
    ev[6].record(s)
    _lib.check_rc(lib.fast_exec(comm._ptr, ctypes.byref(comm.plan.struct),
                                ctypes.c_void_p(send.data_ptr()), e, comm.blocks, comm.chunk,
                                None, sh), "exec")
    ev[7].record(s)
    lib.fast_comm_set_epoch(comm._ptr, e)
    torch.cuda.synchronize()
    if it >= 40:
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(7)]
        # ev[1..4] are gather-end, balance-start/end... per fast_synth_batch_ev:
        # ev1 = start (memset+balance), ev2 = balance end, ev3 = decompose end,
        # ev4 = sort end; ev5 = after synth
        acc += np.array([t[0], t[1], t[2], t[3] + t[4], t[5], t[6],
                         ev[0].elapsed_time(ev[7])])
comm.check()
if rank == 0:
    a = acc / 100 * 1e3
    print(f"{world} GPUs {n}x{m}: " + "  ".join(f"{k} {v:.1f}" for k, v in zip(names, a[:-1]))
          + f"  | total {a[-1]:.1f} us (serialised)", flush=True)
dist.barrier()
for graph in (False, True):
    comm.use_graph = graph
    for _ in range(20):
        comm.alltoallv(send, row)
    torch.cuda.synchronize()
    dist.barrier()
    a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(200):
        comm.alltoallv(send, row)
    b0.record()
    torch.cuda.synchronize()
    if rank == 0:
        print(f"chained call (PDL, graph={graph}): {a0.elapsed_time(b0) / 200 * 1e3:.1f} us", flush=True)
comm.check()
comm.close()
dist.destroy_process_group()
