"""Synthesis time of batches of small matrices for the library in
FASTB200_LIB (A/B of the one-launch small-n kernel).
    python tools/small_batch_ab.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2505_09764_b200 import _lib, synth, workloads  # noqa: E402
lib = _lib.load()
tag = os.path.basename(os.environ.get("FASTB200_LIB", "product"))
for (n, m, B) in [(4, 8, 1000), (6, 8, 1000), (2, 4, 4096), (8, 8, 1000), (12, 8, 1000)]:
    D = workloads.zipf_batch_device(range(B), n*m, 1.2, 1 << 28, "cuda")
    bufs = synth.SynthBuffers(B, n, m)
    s = torch.cuda.current_stream()
    for _ in range(3):
        lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), B, n, m, ctypes.byref(bufs.struct), ctypes.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), B, n, m, ctypes.byref(bufs.struct), ctypes.c_void_p(s.cuda_stream))
    b.record(); torch.cuda.synchronize()
    print(tag, f"n={n} m={m} B={B}: {a.elapsed_time(b)/10*1e3:.1f} us per batch, status max {int(bufs.status.max())}", flush=True)
