"""Tiny-message FastComm calls (for launch-list profiling): 2 ranks needed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist, time
from paper_2505_09764_b200 import Topology, workloads
from paper_2505_09764_b200.executor import FastComm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
D = workloads.gen_hotspot(3, Topology(2, world // 2), 512, hot=0, factor=8).sizes
comm = FastComm(Topology(2, world // 2), recv_bytes=1 << 20, staging_bytes=1 << 20)
send = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
row = torch.from_numpy(D[rank].copy()).cuda()
for _ in range(20): comm.alltoallv(send, row)
torch.cuda.synchronize(); dist.barrier()
for fused, graph in ((True, False), (False, False), (False, True)):
    comm.set_fused(fused)
    comm.use_graph = graph
    for _ in range(20): comm.alltoallv(send, row)
    torch.cuda.synchronize(); dist.barrier()
    t = time.perf_counter()
    for _ in range(200): comm.alltoallv(send, row)
    torch.cuda.synchronize()
    host_us = (time.perf_counter() - t) / 200 * 1e6
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200): comm.alltoallv(send, row)
    b.record(); torch.cuda.synchronize()
    comm.check()
    if rank == 0: print(f"per call (fused={fused}, graph={graph}): wall {host_us:.1f} us, events {a.elapsed_time(b)/200*1e3:.1f} us", flush=True)
comm.close(); dist.destroy_process_group()

# ---- per-stage device breakdown (events between the enqueued stages) ----
import ctypes
from paper_2505_09764_b200 import _lib
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
comm = FastComm(Topology(2, world // 2), recv_bytes=1 << 20, staging_bytes=1 << 20)
lib = _lib.load()
n, m = 2, world // 2
s = torch.cuda.current_stream(); sh = ctypes.c_void_p(s.cuda_stream)
acc = np.zeros(5)
for it in range(120):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    comm.epoch += 1; e = comm.epoch
    ev[0].record(s)
    lib.fast_gather_demand(comm._ptr, ctypes.c_void_p(row.data_ptr()), e, sh); ev[1].record(s)
    dptr = lib.fast_comm_demand_ptr(comm._ptr, e)
    lib.fast_synth_batch(ctypes.c_void_p(dptr), 1, n, m, ctypes.byref(comm.sched.struct), sh); ev[2].record(s)
    lib.fast_plan_compile(ctypes.c_void_p(dptr), ctypes.c_void_p(dptr + 8 * world * world), n, m,
                          ctypes.byref(comm.sched.struct), comm.recv_bytes, comm.staging_bytes,
                          comm.chunk, ctypes.byref(comm.plan.struct), sh); ev[3].record(s)
    lib.fast_exec(comm._ptr, ctypes.byref(comm.plan.struct), ctypes.c_void_p(send.data_ptr()), e,
                  comm.blocks, comm.chunk, None, sh); ev[4].record(s)
    lib.fast_comm_set_epoch(comm._ptr, e)
    torch.cuda.synchronize()
    if it >= 20:
        acc += np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(4)] + [ev[0].elapsed_time(ev[4])])
if rank == 0:
    a = acc / 100 * 1e3
    print(f"stages us: gather {a[0]:.1f}  synth {a[1]:.1f}  plan {a[2]:.1f}  exec {a[3]:.1f}  total {a[4]:.1f}", flush=True)
comm.close(); dist.destroy_process_group()

# ---- fused prologue stamps (globaltimer, ns) ----
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
comm = FastComm(Topology(2, world // 2), recv_bytes=1 << 20, staging_bytes=1 << 20)
acc = np.zeros(7); cnt = 0
for it in range(200):
    comm.alltoallv(send, row, record_timeline=True)
    if it >= 50 and it % 5 == 0:
        t = comm.timeline.cpu().numpy()
        # [5] start, [6] gathered, [7] balanced, [258] decomposed, [0] plan done/barrier start, [1] GO, [3] own ops done, [4] recv complete
        pts = [t[5], t[6], t[7], t[258], t[0], t[3], t[4]]
        acc += np.diff(np.array(pts + [pts[-1]], dtype=np.float64))
        cnt += 1
if rank == 0:
    a = acc / cnt / 1e3
    print(f"fused us: gather {a[0]:.1f} balance {a[1]:.1f} decompose {a[2]:.1f} plan {a[3]:.1f} exec-own {a[4]:.1f} recv-wait {a[5]:.1f}", flush=True)
comm.close(); dist.destroy_process_group()
