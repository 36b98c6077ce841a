"""CPU checks of the compact result layout's host decoders.

The e2e path ships (a) the balanced cross tiles as changed-cell masks +
values and (b) an aux run-out table instead of the per-edge stage bytes
(include/fastb200.h: fast_compact_batch, fast_strip_rec).  Here the compact
form is derived from the ORACLE's full output with an independent encoder
and decoded with the product decoders; the round trip must give the full
layout back bit for bit (and hence the reference's canonical JSON).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from paper_2505_09764_b200 import schedule_to_json, workloads
from paper_2505_09764_b200.schedule import (STRIP_DTYPE, PackedSchedule, balanced_from_compact,
                                            stage_bytes_from_strip)


def encode_tiles(D, bal, n, m):
    masks, vals = [], []
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            a = D[i * m:(i + 1) * m, j * m:(j + 1) * m].ravel()
            b = bal[i * m:(i + 1) * m, j * m:(j + 1) * m].ravel()
            ch = np.flatnonzero(a != b)
            masks.append(int(sum(1 << int(c) for c in ch)))
            vals.extend(b[ch].tolist())
    return np.array(masks, dtype=np.uint64), np.array(vals, dtype=np.int64)


def encode_strip(aux, weight, perm, n):
    recs = np.zeros(2 * n + 2, STRIP_DTYPE)
    recs["stage"] = -1
    slot = 0
    for u in range(n):
        for v in range(n):
            a = int(aux[u, v])
            if a <= 0:
                continue
            left = a
            for k in np.flatnonzero(perm[:, u] == v):
                w = int(weight[k])
                charged = min(left, w)
                left -= charged
                if left == 0:
                    recs[slot] = (w - charged, int(k), u, v)
                    break
            slot += 1
    assert slot <= 2 * n + 2  # the NW-corner staircase bound
    return recs


@pytest.mark.parametrize("n,m,skew,seed", [(3, 2, 0.5, 0), (4, 2, 0.9, 1), (2, 4, 0.3, 2),
                                           (8, 8, 0.8, 3), (16, 8, 0.8, 4), (5, 1, 0.0, 5)])
def test_compact_round_trip_equals_full_layout(n, m, skew, seed):
    D = workloads.zipf_sizes(seed, n * m, skew, 10**9 + seed)
    out = oracle.synthesize_batch(D, n, m)
    full = oracle.packed_fields(out, 0, n, m)
    masks, vals = encode_tiles(D, full["balanced"], n, m)
    bal = balanced_from_compact(D, masks, vals, n, m)
    assert np.array_equal(bal, full["balanced"])
    k = full["n_raw"]
    strip = encode_strip(full["aux"], full["stage_weight"], full["stage_perm"], n)
    sb = stage_bytes_from_strip(full["stage_weight"], full["stage_perm"], strip)
    assert np.array_equal(sb, full["stage_bytes"][:k])
    dec = dict(full, balanced=bal, stage_bytes=sb)
    assert (schedule_to_json(PackedSchedule(**dec).to_schedule())
            == schedule_to_json(PackedSchedule(**full).to_schedule()))


def test_compact_decoder_rejects_a_short_value_list():
    n, m = 2, 2
    D = np.zeros((4, 4), np.int64)
    with pytest.raises(ValueError):
        balanced_from_compact(D, np.array([3, 0], np.uint64), np.array([1], np.int64), n, m)
