"""Where the e2e (host-buffer) config-5 synthesis time goes: per chunk, the
H2D end, synthesis end and fixed-D2H end (CUDA events, ms since the start),
plus the host-side total.  python tools/e2e_timeline.py [chunk] [B] [n]"""
import ctypes, os, sys, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_09764_b200 import _lib, synth, workloads
from paper_2505_09764_b200.synth import _COMPACT_FIELDS

C = int(sys.argv[1]) if len(sys.argv) > 1 else 125
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
n = int(sys.argv[3]) if len(sys.argv) > 3 else 128
m = 8
dev = torch.device("cuda", 0)
D = workloads.zipf_batch_device(range(B), n * m, 0.8, 2**34, dev)
Dh = torch.empty(D.shape, dtype=D.dtype, pin_memory=True)
Dh.copy_(D)
del D
torch.cuda.empty_cache()
hs = synth.HostSchedules(B, n, m)
synth.synthesize_host_batch(Dh, n, m, hs, chunk=C)  # warm
# plain H2D bandwidth of the whole batch (one stream)
Dd = torch.empty(Dh.shape, dtype=Dh.dtype, device=dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); Dd.copy_(Dh, non_blocking=True); b.record(); torch.cuda.synchronize()
print(f"H2D alone: {Dh.numel()*8/1e9:.2f} GB in {a.elapsed_time(b):.1f} ms = "
      f"{Dh.numel()*8/a.elapsed_time(b)/1e6:.1f} GB/s")
out = torch.empty(hs.stage_perm.shape, dtype=torch.uint8, device=dev)
a.record(); hs.stage_perm.copy_(out, non_blocking=True); b.record(); torch.cuda.synchronize()
print(f"D2H alone: {out.numel()/1e9:.2f} GB in {a.elapsed_time(b):.1f} ms = "
      f"{out.numel()/a.elapsed_time(b)/1e6:.1f} GB/s")
del Dd, out
torch.cuda.empty_cache()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    synth.synthesize_host_batch(Dh, n, m, hs, chunk=C)
    el = (time.perf_counter() - t0) * 1e3
    print(f"e2e call {el:.1f} ms -> {B / el * 1e3:.0f} matrices/s; d2h {hs.nbytes()/1e9:.2f} GB")

tr = []
torch.cuda.synchronize()
synth.synthesize_host_batch(Dh, n, m, hs, chunk=C, trace=tr)
torch.cuda.synchronize()
t0 = tr[0]
for kind, i, e in tr[1:]:
    print(f"  chunk {i:2d} {kind:5s} done at {t0.elapsed_time(e):7.1f} ms")

# streaming: depth-2 pipeline over K batches (next batch enqueued before the
# previous one completes)
K = 4
pipe = synth.HostSynthPipeline(B, n, m, chunk=C, depth=2)
outs = [hs, synth.HostSchedules(B, n, m)]
pipe.run([Dh] * 2, outs)  # warm (sizes the value buffers)
torch.cuda.synchronize()
t0 = time.perf_counter()
pipe.run([Dh] * K, [outs[k % 2] for k in range(K)])
el = (time.perf_counter() - t0) * 1e3
print(f"streaming depth 2: {K} batches in {el:.1f} ms -> {K * B / el * 1e3:.0f} matrices/s")
