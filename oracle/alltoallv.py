"""CPU ORACLE for the data path -- test infrastructure only.

The reference (tiersched) moves no bytes: its executor is the
analytical simulate_fast (simulate.py:107-193).  The byte-level contract of
the B200 executor is therefore the plain alltoallv it implements:

    recv_h[seg g] = send_g[seg h]

with send_g's segment for h at offset sum_{h'<h} D[g,h'] and recv_h's
segment from g at offset sum_{g'<g} D[g',h]; self traffic (diagonal) is zero
and handled out of band.  This module restates that
contract in numpy, plus deterministic payload bytes (SplitMix64 stream
0xFA57_0000 + g, little-endian -- SURVEY.md 8(d)).
"""

from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
PAYLOAD_SEED = 0xFA57_0000


def splitmix_stream(seed: int, count: int) -> np.ndarray:
    k = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        return z ^ (z >> np.uint64(31))


def payload(rank: int, nbytes: int) -> np.ndarray:
    """Send-buffer bytes of GPU `rank`: little-endian SplitMix64 words."""
    words = splitmix_stream(PAYLOAD_SEED + rank, (nbytes + 7) // 8)
    return words.view(np.uint8)[:nbytes].copy()


def direct_alltoallv(sends: list[np.ndarray], D: np.ndarray) -> list[np.ndarray]:
    """recv_h = concat over g of send_g[off_g(h) : off_g(h) + D[g,h]]."""
    G = D.shape[0]
    send_off = np.concatenate([np.zeros((G, 1), np.int64), np.cumsum(D, axis=1)[:, :-1]], axis=1)
    out = []
    for h in range(G):
        parts = [sends[g][send_off[g, h]:send_off[g, h] + D[g, h]] for g in range(G)]
        out.append(np.concatenate(parts) if parts else np.zeros(0, np.uint8))
    return out
