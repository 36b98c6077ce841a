"""Run the batched synthesis a few times (for ncu / timing experiments).

    python tools/profile_synth.py --n 128 --batch 148 --reps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2505_09764_b200 import synth, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--batch", type=int, default=148)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--skew", type=float, default=0.8)
ap.add_argument("--compact", action="store_true", help="also the strip table + compact pack")
a = ap.parse_args()
D = workloads.zipf_batch_device(range(a.batch), a.n * a.m, a.skew, 2**34, "cuda")
bufs = synth.SynthBuffers(a.batch, a.n, a.m, compact=a.compact)
if a.compact:
    import ctypes
    from paper_2505_09764_b200 import _lib
    lib = _lib.load()
    T = a.n * (a.n - 1)
    vals = torch.empty(a.batch * T * a.m * a.m, dtype=torch.int64, device="cuda")
    base = torch.empty(a.batch + 1, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(lib.fast_compact_workspace_bytes(a.batch)), dtype=torch.uint8, device="cuda")
for r in range(a.reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    synth.synthesize_packed(D, a.n, a.m, bufs)
    if a.compact:
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check_rc(lib.fast_compact_batch(ctypes.byref(bufs.struct), a.batch, a.n, a.m, P(vals),
                                             P(base), P(ws), None), "compact")
    e.record()
    torch.cuda.synchronize()
    print(f"rep {r}: {s.elapsed_time(e):.3f} ms, status max {int(bufs.status.max())}", flush=True)
