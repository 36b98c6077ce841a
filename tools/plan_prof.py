"""Phase timings of the CTA-parallel device plan (needs a -DFAST_PLAN_PROFILE
build: FASTB200_LIB=paper_2505_09764_b200/libfastb200_prof.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_09764_b200 import _lib, synth, workloads  # noqa: E402
from paper_2505_09764_b200.executor import PlanBuffers  # noqa: E402

lib = _lib.load()
lib.fast_debug_plan_prof.argtypes = [ctypes.c_void_p]
names = ["entry->status", "stage inputs", "P1+P2", "take scan", "P3", "P4 count", "P5+scan",
         "P6 emit", "status"]
for n, m in [(2, 1), (2, 2), (2, 4), (4, 2), (8, 1)]:
    G = n * m
    D = torch.from_numpy(workloads.zipf_sizes(1, G, 1.2, 1 << 26)).cuda().view(1, G, G)
    sb = torch.zeros(G, dtype=torch.int64, device="cuda")
    bufs = synth.SynthBuffers(1, n, m)
    plan = PlanBuffers(n, m, "cuda")
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), 1, n, m, ctypes.byref(bufs.struct), sh)
    acc = np.zeros(9)
    for it in range(20):
        lib.fast_plan_compile(ctypes.c_void_p(D.data_ptr()), ctypes.c_void_p(sb.data_ptr()), n, m,
                              ctypes.byref(bufs.struct), 1 << 30, 1 << 30, 1 << 20,
                              ctypes.byref(plan.struct), sh)
        torch.cuda.synchronize()
        out = (ctypes.c_longlong * 16)()
        lib.fast_debug_plan_prof(out)
        st = [out[9]] + [out[k] for k in range(9)]
        if it >= 5:
            acc += np.diff(np.array(st, dtype=np.float64))
    acc /= 15
    print(f"{n}x{m} ops {int(plan.n_ops.item())} total {acc.sum():.0f} cyc: " +
          ", ".join(f"{nm} {v:.0f}" for nm, v in zip(names, acc)), flush=True)
