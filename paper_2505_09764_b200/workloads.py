"""Seeded synthetic inputs: SplitMix64 stream and demand-matrix generators.

Restates tiersched.rng (rng.py:1-49) and tiersched.workloads
(workloads.py:16-85) so that the same (seed, topology, parameters) produce
the same matrices.  One deliberate extension: ``gen_zipf`` accepts skew >= 1
(BASELINE config 2 uses alpha = 1.2; the reference rejects it at
workloads.py:41-42).  For skew < 1 the output is identical to the
reference's (tests/test_workloads.py).  These generators build benchmark
inputs on the host; they are not part of the timed path.
"""

from __future__ import annotations

import numpy as np

from .model import DemandMatrix, Topology, ValidationError

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


def mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def stream(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Outputs offset..offset+count-1: mix64(seed + (k+1)*GOLDEN) as uint64."""
    if count < 0:
        raise ValueError("count must be non-negative")
    k = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + k * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        return z ^ (z >> np.uint64(31))


def value(seed: int, index: int) -> int:
    return mix64((seed + (index + 1) * GOLDEN) & MASK64)


def gen_uniform(seed: int, t: Topology, mean_bytes: int) -> DemandMatrix:
    """Uniform on [0, 2*mean] per off-diagonal pair (workloads.py:16-27)."""
    mean_bytes = int(mean_bytes)
    if mean_bytes <= 0:
        raise ValidationError("mean_bytes must be positive")
    g = t.gpu_count
    sizes = (stream(seed, g * g) % np.uint64(2 * mean_bytes + 1)).astype(np.int64).reshape(g, g)
    np.fill_diagonal(sizes, 0)
    return DemandMatrix(t.n_servers, t.gpus_per_server, sizes)


def zipf_sizes(seed: int, g: int, skew: float, total_bytes: int) -> np.ndarray:
    """Zipf shares over a seeded pair ranking with an exact total
    (workloads.py:44-62), any skew >= 0."""
    pairs = g * g - g
    order = np.argsort(stream(seed, pairs), kind="stable")
    ranks = np.arange(1, pairs + 1, dtype=np.float64)
    weights = 1.0 / ranks ** skew
    shares = total_bytes * weights / weights.sum()
    base = np.floor(shares).astype(np.int64)
    leftover = total_bytes - int(base.sum())
    if leftover > 0:
        frac = shares - base
        base[np.lexsort((np.arange(pairs), -frac))[:leftover]] += 1
    sizes = np.zeros((g, g), dtype=np.int64)
    offdiag = np.flatnonzero(~np.eye(g, dtype=bool).ravel())
    sizes.ravel()[offdiag[order]] = base
    return sizes


def _zipf_base(pairs: int, skew: float, total_bytes: int) -> np.ndarray:
    """Rank-ordered integer shares; independent of the seed."""
    ranks = np.arange(1, pairs + 1, dtype=np.float64)
    weights = 1.0 / ranks ** skew
    shares = total_bytes * weights / weights.sum()
    base = np.floor(shares).astype(np.int64)
    leftover = total_bytes - int(base.sum())
    if leftover > 0:
        frac = shares - base
        base[np.lexsort((np.arange(pairs), -frac))[:leftover]] += 1
    return base


def _s64(x: int) -> int:
    return x - (1 << 64) if x >= 1 << 63 else x


def stream_device(seeds, count: int, device):
    """SplitMix64 outputs 0..count-1 for each seed, as int64 bit patterns
    (torch int64 arithmetic wraps like uint64; shifts are made logical)."""
    import torch

    s = torch.as_tensor([_s64(int(x) & MASK64) for x in seeds], dtype=torch.int64,
                        device=device)[:, None]
    k = torch.arange(1, count + 1, dtype=torch.int64, device=device)[None, :]
    z = s + k * _s64(GOLDEN)
    z = (z ^ ((z >> 30) & ((1 << 34) - 1))) * _s64(MIX1)
    z = (z ^ ((z >> 27) & ((1 << 37) - 1))) * _s64(MIX2)
    return z ^ ((z >> 31) & ((1 << 33) - 1))


def zipf_batch_device(seeds, g: int, skew: float, total_bytes: int, device, chunk: int = 32):
    """[len(seeds), g, g] int64 on ``device``; equal to stacking
    ``zipf_sizes(seed, g, skew, total_bytes)`` (the base shares do not depend
    on the seed, only the stable argsort of the seed's stream does)."""
    import torch

    pairs = g * g - g
    base = torch.from_numpy(_zipf_base(pairs, skew, int(total_bytes))).to(device)
    offdiag = torch.from_numpy(np.flatnonzero(~np.eye(g, dtype=bool).ravel())).to(device)
    seeds = list(seeds)
    out = torch.zeros((len(seeds), g * g), dtype=torch.int64, device=device)
    for c0 in range(0, len(seeds), chunk):
        cs = seeds[c0:c0 + chunk]
        keys = stream_device(cs, pairs, device) ^ _s64(1 << 63)  # unsigned order
        order = torch.sort(keys, dim=1, stable=True).indices
        out[c0:c0 + len(cs)].scatter_(1, offdiag[order], base.expand(len(cs), pairs))
    return out.view(len(seeds), g, g)


def gen_zipf(seed: int, t: Topology, skew: float, total_bytes: int) -> DemandMatrix:
    if not skew >= 0.0:
        raise ValidationError("skew must be >= 0")
    total_bytes = int(total_bytes)
    if total_bytes <= 0:
        raise ValidationError("total_bytes must be positive")
    return DemandMatrix(t.n_servers, t.gpus_per_server,
                        zipf_sizes(seed, t.gpu_count, skew, total_bytes))


def gen_adversarial(t: Topology, tile_bytes: int) -> DemandMatrix:
    """GPU 0 of every server sends tile_bytes to GPU 0 of every other one."""
    tile_bytes = int(tile_bytes)
    if tile_bytes <= 0:
        raise ValidationError("tile_bytes must be positive")
    n, m = t.n_servers, t.gpus_per_server
    sizes = np.zeros((t.gpu_count, t.gpu_count), dtype=np.int64)
    for i in range(n):
        for j in range(n):
            if i != j:
                sizes[i * m, j * m] = tile_bytes
    return DemandMatrix(n, m, sizes)


def gen_hotspot(seed: int, t: Topology, mean_bytes: int, hot: int, factor: int) -> DemandMatrix:
    """Config 4: uniform base with GPU ``hot``'s row and column scaled x factor."""
    d = gen_uniform(seed, t, mean_bytes).sizes.copy()
    d[hot, :] *= factor
    d[:, hot] *= factor
    np.fill_diagonal(d, 0)
    return DemandMatrix(t.n_servers, t.gpus_per_server, d)


def load_trace(path: str) -> DemandMatrix:
    """Load a demand matrix from a JSON or CSV trace file (workloads.py:88-90)."""
    from .model import load_matrix

    return load_matrix(path)
