"""Pin the CPU oracle (oracle/fast_oracle.c) to the reference.

Every golden fixture was produced by tiersched itself (tests/golden/
make_golden.py); the oracle must reproduce each canonical schedule JSON byte
for byte, and each decomposition (aux, raw stages, stripped+sorted stages).
When /root/reference is present a live comparison on fresh seeds runs too.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import import_reference, reference_available
from oracle import oracle
from paper_2505_09764_b200.schedule import PackedSchedule, schedule_to_json


def oracle_json(D: np.ndarray, n: int, m: int) -> str:
    out = oracle.synthesize_batch(D, n, m)
    assert int(out["status"][0]) == 0
    return schedule_to_json(PackedSchedule(**oracle.packed_fields(out, 0, n, m)).to_schedule())


def test_oracle_matches_every_golden_schedule(golden_schedules):
    assert len(golden_schedules) >= 300
    for rec in golden_schedules:
        D = np.array(rec["D"], dtype=np.int64)
        got = oracle_json(D, rec["n"], rec["m"])
        assert got == rec["json"], rec["name"]


def _stages(out, k_idx, n, use_bytes):
    res = []
    for k in k_idx:
        w = int(out["stage_weight"][k])
        if use_bytes:
            row = out["stage_bytes"][k]
            edges = [[u, int(out["stage_perm"][k][u]), int(row[u])] for u in range(n) if row[u] > 0]
        else:
            edges = [[u, int(out["stage_perm"][k][u]), w] for u in range(n)]
        res.append([w, edges])
    return res


def test_oracle_matches_every_golden_decomposition(golden_decompositions):
    for rec in golden_decompositions:
        S = np.array(rec["S"], dtype=np.int64)
        n = S.shape[0]
        out = oracle.decompose_server(S)
        assert out["status"] == 0, rec["name"]
        assert int(out["common_sum"][0]) == rec["common_sum"], rec["name"]
        assert out["aux"].tolist() == rec["aux"], rec["name"]
        k = int(out["n_raw"][0])
        assert _stages(out, range(k), n, False) == rec["raw"], rec["name"]
        order = out["stage_order"][: int(out["n_stages"][0])]
        assert _stages(out, order, n, True) == rec["sorted"], rec["name"]


def test_oracle_validation_errors():
    D = np.zeros((4, 4), np.int64)
    D[0, 0] = 1
    assert int(oracle.synthesize_batch(D, 2, 2)["status"][0]) == 2
    D = np.zeros((4, 4), np.int64)
    D[0, 1] = -1
    assert int(oracle.synthesize_batch(D, 2, 2)["status"][0]) == 2
    D = np.zeros((4, 4), np.int64)
    D[0, 2] = 1 << 61
    D[1, 3] = 1 << 61
    assert int(oracle.synthesize_batch(D, 2, 2)["status"][0]) == 2
    D[1, 3] -= 1
    assert int(oracle.synthesize_batch(D, 2, 2)["status"][0]) == 0


@pytest.mark.skipif(not reference_available(), reason="reference tree not mounted")
def test_oracle_live_against_reference():
    ts = import_reference()
    rng = np.random.default_rng(1234)
    for trial in range(60):
        n = int(rng.integers(2, 9))
        m = int(rng.integers(1, 6))
        t = ts.Topology(n, m, 900e9, 900e9)
        kind = trial % 3
        if kind == 0:
            d = ts.gen_uniform(trial, t, int(rng.integers(1, 10**6)))
        elif kind == 1:
            d = ts.gen_zipf(trial, t, float(rng.uniform(0, 0.99)), int(rng.integers(1, 10**12)))
        else:  # sparse: many zeros, exercises empty stages / aux on the diagonal
            s = ts.gen_uniform(trial, t, 50).sizes
            s[rng.random(s.shape) < 0.7] = 0
            d = ts.DemandMatrix(n, m, s)
        want = ts.schedule_to_json(ts.synthesize_fast(d, t))
        assert oracle_json(d.sizes, n, m) == want, (trial, n, m)
