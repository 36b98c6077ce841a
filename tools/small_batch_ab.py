import ctypes, os, sys
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.getcwd())
import torch
from paper_2505_09764_b200 import _lib, synth, workloads
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
