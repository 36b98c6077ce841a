"""Balance-kernel A/B on config 5: device time of fast_balance_batch (CUDA
events, best of reps) for each library given, and bit-equality of every
output (balanced, server, moves, move counts, tile masks, status) against
the first library.

    python tools/bal_ab.py LIB_A.so [LIB_B.so ...]   (env N, M, B, REPS)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_09764_b200 import synth, workloads  # noqa: E402

n = int(os.environ.get("N", 128))
m = int(os.environ.get("M", 8))
B = int(os.environ.get("B", 1000))
reps = int(os.environ.get("REPS", 5))
dev = torch.device("cuda", 0)
D = workloads.zipf_batch_device(range(B), n * m, float(os.environ.get("SKEW", 0.8)), 2**34, dev)
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
bufs = synth.SynthBuffers(B, n, m, dev, stage_bytes=False, compact=True)
G = n * m
alg = 16 * G * G * B
ref = None
for path in sys.argv[1:]:
    lib = ctypes.CDLL(path)
    lib.fast_balance_batch.restype = ctypes.c_int
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for r in range(reps + 1):
        bufs.balanced.fill_(-7)
        ev[0].record(s)
        rc = lib.fast_balance_batch(ctypes.c_void_p(D.data_ptr()), B, n, m,
                                    ctypes.byref(bufs.struct), sh)
        ev[1].record(s)
        torch.cuda.synchronize()
        assert rc == 0, rc
        if r:
            ts.append(ev[0].elapsed_time(ev[1]))
    T = n * (n - 1)
    outs = {
        "balanced": bufs.balanced.clone(),
        "server": bufs.server.clone(),
        "move_count": bufs.move_count.clone(),
        "moves": bufs.moves.clone(),
        "tile_mask": bufs.tile_mask.clone(),
        "status": bufs.status.clone(),
    }
    same = ""
    if ref is None:
        ref = outs
    else:
        # moves beyond each tile's count are unspecified: compare used slots only
        mc = outs["move_count"].view(B * T).long()
        slots = max(m - 1, 1)
        used = (torch.arange(slots, device=dev)[None, :] < mc[:, None]).reshape(-1)
        bad = []
        for k, v in outs.items():
            a, b = v, ref[k]
            if k == "moves":
                a = a.view(B * T * slots, -1)[used]
                b = b.view(B * T * slots, -1)[used]
            if not torch.equal(a, b):
                bad.append(k)
        same = "bit-equal" if not bad else f"DIFFERS in {bad}"
    best = min(ts)
    print(f"{os.path.basename(path)}: balance {best:.3f} ms (median {sorted(ts)[len(ts)//2]:.3f}) "
          f"{alg / best / 1e6:.0f} GB/s alg, status max {int(outs['status'].max())} {same}", flush=True)
