"""CPU ORACLE for the MoE dispatch front-end -- test infrastructure only.

The reference has no MoE front-end; this restates the recipe
of SURVEY.md 8(d) config 3 in numpy:
  * gating: w_e = 1/((e - hot) mod E + 1)^alpha; integer CDF thresholds
    thr = floor(cumsum(w)/sum(w) * 2^32), thr[E-1] = 2^32; for source s,
    r = stream(seed*1000 + s, 2T) >> 32, e1 = searchsorted(thr, r[:T],
    'right'), e2 = searchsorted(thr2[e1], r[T:], 'right') with thr2[e] the
    thresholds of w with w[e] = 0;
  * counts[s] = bincount(e1) + bincount(e2); D row = counts * row_bytes;
  * pack: destination segments in expert order, tokens in ascending order;
  * expert input on GPU h: source-major concat of every source's segment h.
"""

from __future__ import annotations

import numpy as np

from oracle.alltoallv import splitmix_stream


def thresholds(E: int, alpha: float = 0.8, hot: int = 0) -> tuple[np.ndarray, np.ndarray]:
    w = 1.0 / (((np.arange(E) - hot) % E) + 1.0) ** alpha

    def cdf(x):
        t = np.floor(np.cumsum(x) / x.sum() * 2.0 ** 32).astype(np.uint64)
        t[-1] = np.uint64(1 << 32)
        return t

    thr2 = np.stack([cdf(np.where(np.arange(E) == e, 0.0, w)) for e in range(E)])
    return cdf(w), thr2


def gate(seed: int, src: int, T: int, thr: np.ndarray, thr2: np.ndarray) -> np.ndarray:
    r = splitmix_stream(seed * 1000 + src, 2 * T) >> np.uint64(32)
    e1 = np.searchsorted(thr, r[:T], side="right")
    e2 = (thr2[e1] <= r[T:, None]).sum(axis=1)
    return np.stack([e1, e2], axis=1).astype(np.int32)


def route(topk: np.ndarray, E: int):
    flat = topk.reshape(-1)
    counts = np.bincount(flat, minlength=E).astype(np.int64)
    seg = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    order = np.argsort(flat, kind="stable")  # entries grouped by expert, token order
    return counts, seg, order


def pack(tokens: np.ndarray, topk: np.ndarray, E: int) -> np.ndarray:
    """tokens [T, row_bytes] uint8 -> send rows [T*k, row_bytes]."""
    _, _, order = route(topk, E)
    k = topk.shape[1]
    return tokens[order // k]


def expert_inputs(tokens: list[np.ndarray], topks: list[np.ndarray], E: int,
                  experts_per_rank: int = 1) -> list[np.ndarray]:
    """Expert input rows of every GPU h (source-major, self included; within
    a source, GPU h's experts h*L .. h*L+L-1 in order, tokens ascending)."""
    G, L = len(tokens), experts_per_rank
    sends = [pack(tokens[s], topks[s], E) for s in range(G)]
    segs = [route(topks[s], E) for s in range(G)]
    out = []
    for h in range(G):
        parts = []
        for s in range(G):
            counts, seg, _ = segs[s]
            a = seg[h * L]
            b = seg[h * L + L - 1] + counts[h * L + L - 1]
            parts.append(sends[s][a:b])
        out.append(np.concatenate(parts))
    return out


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16(f: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even (finite inputs)."""
    b = f.astype(np.float32).view(np.uint32)
    return ((b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def combine(tokens_bf16: list[np.ndarray], topks: list[np.ndarray], weights: list[np.ndarray],
            expert_scale) -> list[np.ndarray]:
    """out[t] = bf16( sum_j fl32(w[t,j] * x_j) ) accumulated left to right in
    float32 (IEEE round-to-nearest per op), x_j = expert e_j's output for
    token t = token * expert_scale(e_j) (exact power-of-two scaling)."""
    outs = []
    for s in range(len(tokens_bf16)):
        x = bf16_to_f32(tokens_bf16[s])  # [T, H]
        tk, w = topks[s], weights[s].astype(np.float32)
        acc = None
        for j in range(tk.shape[1]):
            scale = np.array([expert_scale(int(e)) for e in tk[:, j]], np.float32)[:, None]
            xj = (x * scale).astype(np.float32)
            p = (w[:, j:j + 1] * xj).astype(np.float32)
            acc = p if acc is None else (acc + p).astype(np.float32)
        outs.append(f32_to_bf16(acc))
    return outs
