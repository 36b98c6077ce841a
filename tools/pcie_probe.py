"""PCIe copy bandwidth on the GPU box: pinned H2D alone, D2H alone, and both
directions at once on separate streams (the e2e pipeline's situation), plus
the H2D rate when D2H runs at the e2e ratio (5.88 GB back per 8.39 GB in).

    python tools/pcie_probe.py [GB]
"""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
n = int(gb * 2**30) // 8
dev = torch.device("cuda", 0)
h_in = torch.empty(n, dtype=torch.int64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.int64, pin_memory=True)
d_in = torch.empty(n, dtype=torch.int64, device=dev)
d_out = torch.empty(n, dtype=torch.int64, device=dev)
h_in.fill_(1)
d_out.fill_(2)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h(k=n):
    with torch.cuda.stream(s2):
        h_out[:k].copy_(d_out[:k], non_blocking=True)


def both(k=n):
    h2d()
    d2h(k)


B = n * 8 / 1e9
t = timed(h2d)
print(f"H2D alone: {B:.2f} GB in {t*1e3:.1f} ms = {B/t:.1f} GB/s")
t = timed(d2h)
print(f"D2H alone: {B:.2f} GB in {t*1e3:.1f} ms = {B/t:.1f} GB/s")
t = timed(both)
print(f"H2D + D2H concurrently: 2 x {B:.2f} GB in {t*1e3:.1f} ms = {2*B/t:.1f} GB/s aggregate")
k = int(n * 5.88 / 8.39)
t = timed(lambda: both(k))
print(f"H2D {B:.2f} GB + D2H {k*8/1e9:.2f} GB (e2e ratio) concurrently: {t*1e3:.1f} ms "
      f"(H2D alone would take {B/ (B/timed(h2d)) * 1e3:.1f} ms)")
# chunked: 8 chunks per direction, interleaved on 8 streams each way
streams = [torch.cuda.Stream(dev) for _ in range(16)]


def chunked():
    c = n // 8
    for i in range(8):
        with torch.cuda.stream(streams[i]):
            d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(streams[8 + i]):
            kk = int(c * 5.88 / 8.39)
            h_out[i * c:i * c + kk].copy_(d_out[i * c:i * c + kk], non_blocking=True)


t = timed(chunked)
print(f"8-chunk H2D {B:.2f} GB + D2H at the e2e ratio, 16 streams: {t*1e3:.1f} ms")
