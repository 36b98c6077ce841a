"""Decompose-kernel A/B on config 5: per-kernel device time (CUDA events)
for the full (per-edge stage bytes) and compact (strip table) output modes,
for the library in FASTB200_LIB (default: in-tree build).

    python tools/dec_ab.py [n] [B] [reps]
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_09764_b200 import _lib, synth, workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m = 8
lib = _lib.load()
dev = torch.device("cuda", 0)
D = workloads.zipf_batch_device(range(B), n * m, 0.8, 2**34, dev)
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
tag = os.path.basename(os.environ.get("FASTB200_LIB", "default"))
for mode in os.environ.get("MODES", "full,compact").split(","):
    bufs = synth.SynthBuffers(B, n, m, dev, stage_bytes=(mode == "full"), compact=(mode == "compact"))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record(s)
    arr = (ctypes.c_void_p * 4)(*[e.cuda_event for e in ev])
    res = []
    for r in range(reps + 1):
        _lib.check_rc(lib.fast_synth_batch_ev(ctypes.c_void_p(D.data_ptr()), B, n, m,
                                              ctypes.byref(bufs.struct), sh, arr), "synth")
        torch.cuda.synchronize()
        if r:
            res.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
    st = int(bufs.status.abs().max())
    best = [min(x[i] for x in res) for i in range(3)]
    print(f"{tag} {mode:8s} n={n} B={B}: balance {best[0]:.3f} decompose {best[1]:.3f} "
          f"sort {best[2]:.3f} ms status {st}", flush=True)
    del bufs
    torch.cuda.empty_cache()
