"""Section timings of decompose_kernel (needs a -DFAST_DEC_PROFILE build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_09764_b200 import _lib, synth, workloads
n, B = int(sys.argv[1]), int(sys.argv[2])
lib = _lib.load()
D = workloads.zipf_batch_device(range(B), n * 8, 0.8, 2**34, "cuda")
bufs = synth.SynthBuffers(B, n, 8)
synth.synthesize_packed(D, n, 8, bufs)
out = (ctypes.c_ulonglong * 8)()
lib.fast_debug_dec_prof(out, 1)
s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record(); synth.synthesize_packed(D, n, 8, bufs); e0.record(); torch.cuda.synchronize()
lib.fast_debug_dec_prof(out, 1)
head, dfs, app, mov, steps, peels = out[0], out[1], out[2], out[3], out[4], out[5]
tot = head + dfs + app + mov
print(f"n={n} B={B} time {s0.elapsed_time(e0):.1f} ms; per matrix: peels {peels/B:.0f}, dfs steps {steps/B:.0f}")
for name, v in [("head(min/subtract/stage out)", head), ("dfs", dfs), ("apply_path", app), ("moved rows", mov)]:
    print(f"  {name:30s} {v/tot*100:5.1f}%  {v/peels:8.0f} cyc/peel")
print(f"  dfs cycles/step {dfs/steps:.0f}; total cycles/peel {tot/peels:.0f}")
