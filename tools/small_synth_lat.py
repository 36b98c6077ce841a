"""Single-matrix synthesis latency (B=1, device time per call from a CUDA
graph of back-to-back calls) at the BASELINE small shapes, for the library
in FASTB200_LIB.   python tools/small_synth_lat.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_09764_b200 import _lib, synth, workloads  # noqa: E402

lib = _lib.load()
tag = os.path.basename(os.environ.get("FASTB200_LIB", "product"))
res = []
for n, m in [(2, 1), (2, 2), (4, 1), (2, 4), (4, 2), (4, 8), (6, 8), (8, 8), (10, 8), (12, 8), (12, 4), (16, 8)]:
    D = torch.from_numpy(workloads.zipf_sizes(0, n * m, 1.2, 1 << 28)).cuda().view(1, n * m, n * m)
    bufs = synth.SynthBuffers(1, n, m)
    s = torch.cuda.Stream()
    calls = 50
    with torch.cuda.stream(s):
        for _ in range(3):
            _lib.check_rc(lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), 1, n, m,
                                               ctypes.byref(bufs.struct), ctypes.c_void_p(s.cuda_stream)), "w")
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(calls):
            lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), 1, n, m, ctypes.byref(bufs.struct),
                                 ctypes.c_void_p(s.cuda_stream))
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / calls * 1e3)
    assert int(bufs.status.item()) == 0
    res.append(f"{n}x{m} {best:.1f}")
print(tag + ": " + "  ".join(res) + "  (us per call)", flush=True)
