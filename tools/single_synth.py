"""Device latency of the per-call synthesis pieces for one small matrix."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_09764_b200 import _lib, synth, workloads
from paper_2505_09764_b200.executor import PlanBuffers
lib = _lib.load()
s = torch.cuda.current_stream(); sh = ctypes.c_void_p(s.cuda_stream)
shapes = [(2, 1), (2, 2), (2, 4), (4, 2)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split('x')) for a in sys.argv[1:]]
for n, m in shapes:
    G = n * m
    D = torch.from_numpy(workloads.zipf_sizes(1, G, 1.2, 1 << 26)).cuda().view(1, G, G)
    self_b = torch.zeros(G, dtype=torch.int64, device="cuda")
    bufs = synth.SynthBuffers(1, n, m)
    plan = PlanBuffers(n, m, "cuda")
    def run(k):
        sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        if k in (0, 2):
            lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), 1, n, m, ctypes.byref(bufs.struct), sh)
        if k in (1, 2):
            lib.fast_plan_compile(ctypes.c_void_p(D.data_ptr()), ctypes.c_void_p(self_b.data_ptr()), n, m,
                                  ctypes.byref(bufs.struct), 1 << 30, 1 << 30, 1 << 20, ctypes.byref(plan.struct), sh)
    out = []
    for k in range(3):
        for _ in range(20): run(k)
        torch.cuda.synchronize()
        # graph of 50 back-to-back calls: device time without host launch gaps
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(50): run(k)
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / 50 * 1e3)
    print(f"{n}x{m}: synth {out[0]:.1f} us  plan {out[1]:.1f} us  synth+plan {out[2]:.1f} us  (ops {int(plan.n_ops.item())})", flush=True)
