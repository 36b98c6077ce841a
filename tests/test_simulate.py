"""Analytical cost model (simulate_fast / simulate_spreadout / bounds).

CPU: the oracle restatement (oracle/simulate.py) is pinned bit for bit to the
reference's own outputs (tests/golden/simulate.json.gz, made by
tests/golden/make_sim_golden.py from tiersched).  GPU: the batched sm_100a
simulator (csrc/sim.cu) through the C-ABI and through the drop-in object API
(simulate_fast(plan, stages, t)) equals the same fixtures bit for bit.
"""

from __future__ import annotations

import gzip
import json
import os

import numpy as np
import pytest

from conftest import REPO
from oracle import oracle
from oracle import simulate as sim_oracle

GOLDEN = os.path.join(REPO, "tests", "golden", "simulate.json.gz")


def _golden():
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)


def _f(h: str) -> float:
    return float.fromhex(h)


def _hex(xs):
    return [float(x).hex() for x in xs]


def test_oracle_matches_reference_fixtures():
    rows = _golden()
    assert len(rows) >= 100
    for r in rows:
        n, m = r["n"], r["m"]
        b1, b2, a = (_f(x) for x in r["topo"])
        D = np.array(r["sizes"], dtype=np.int64)
        out = oracle.synthesize_batch(D, n, m)
        p = oracle.packed_fields(out, 0, n, m)
        got = sim_oracle.simulate_fast(p, b1, b2, a)
        want = r["fast"]
        assert "error" not in got, r["name"]
        assert float(got["t_balance"]).hex() == want["t_balance"], r["name"]
        assert float(got["t_intra_a2a"]).hex() == want["t_intra_a2a"], r["name"]
        assert _hex(got["scale_out"]) == want["scale_out"], r["name"]
        assert _hex(got["redistribution"]) == want["redistribution"], r["name"]
        assert float(got["total"]).hex() == want["total"], r["name"]
        server = np.asarray(p["server"], dtype=np.int64)
        so = sim_oracle.simulate_spreadout(server, m, b2, a)
        assert _hex(so["scale_out"]) == r["spreadout"]["scale_out"], r["name"]
        assert float(so["total"]).hex() == r["spreadout"]["total"], r["name"]
        sod = sim_oracle.simulate_spreadout(server, m, b2, a, demand=D)
        assert _hex(sod["scale_out"]) == r["spreadout_demand"]["scale_out"], r["name"]
        assert float(sod["total"]).hex() == r["spreadout_demand"]["total"], r["name"]
        assert sim_oracle.spreadout_weights(server) == r["spreadout_weights"]
        bd = sim_oracle.bounds(server, m, b1, b2)
        assert float(bd["t_optimal"]).hex() == r["t_optimal"], r["name"]
        assert float(bd["t_worstcase"]).hex() == r["t_worstcase"], r["name"]
        assert float(bd["ratio_bound"]).hex() == r["ratio_bound"], r["name"]
        assert bd["assumption_ok"] == r["assumption_ok"], r["name"]


def test_fixture_exercises_the_exact_integer_split():
    # split_deliveries switches to exact integers when cell * r >= 2^63
    # (balance.py:196-199); the "huge" instances must reach that branch
    hit = 0
    for r in _golden():
        if not r["name"].startswith("huge"):
            continue
        D = np.array(r["sizes"], dtype=np.int64)
        hit += int(D.max()) * int(D.max()) >= (1 << 63)
    assert hit >= 5


def test_hand_checked_kat():
    # test_simulate.py:105-122 of the reference: one swap stage of weight 60
    r = [x for x in _golden() if x["name"] == "kat_2x1"][0]
    assert [_f(x) for x in r["fast"]["scale_out"]] == [0.5 + 60 / 10.0]
    assert _f(r["fast"]["t_balance"]) == 0.0 and _f(r["fast"]["t_intra_a2a"]) == 0.0


def _check_fields(got: dict, r: dict, S: int):
    want = r["fast"]
    assert float(got["t_balance"]).hex() == want["t_balance"], r["name"]
    assert float(got["t_intra"]).hex() == want["t_intra_a2a"], r["name"]
    assert _hex(got["scale_out"][:S]) == want["scale_out"], r["name"]
    assert _hex(got["redistribution"][:S]) == want["redistribution"], r["name"]
    assert float(got["total"]).hex() == want["total"], r["name"]
    n = r["n"]
    assert _hex(got["so_server"][: n - 1]) == r["spreadout"]["scale_out"], r["name"]
    assert float(got["so_total"][0]).hex() == r["spreadout"]["total"], r["name"]
    assert _hex(got["so_demand"][: n - 1]) == r["spreadout_demand"]["scale_out"], r["name"]
    assert float(got["so_total"][1]).hex() == r["spreadout_demand"]["total"], r["name"]
    assert [int(x) for x in got["so_weight"][: n - 1]] == r["spreadout_weights"], r["name"]
    assert float(got["t_optimal"]).hex() == r["t_optimal"], r["name"]
    assert float(got["t_worstcase"]).hex() == r["t_worstcase"], r["name"]
    assert bool(got["assumption_ok"]) == r["assumption_ok"], r["name"]


@pytest.mark.gpu
def test_batched_device_model_matches_reference():
    """Device synthesis -> fast_simulate_batch on the device output, whole
    batches per topology, every field bit-identical to the reference."""
    import torch

    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.simulate import simulate_batch
    from paper_2505_09764_b200.synth import synthesize_packed

    groups: dict = {}
    for r in _golden():
        groups.setdefault((r["n"], r["m"], tuple(r["topo"])), []).append(r)
    for (n, m, topo), rows in groups.items():
        b1, b2, a = (_f(x) for x in topo)
        t = Topology(n, m, scaleup_bw=b1, scaleout_bw=b2, wakeup_delay=a)
        D = torch.tensor(np.stack([np.array(r["sizes"], np.int64) for r in rows])).cuda()
        bufs = synthesize_packed(D, n, m)
        out = simulate_batch(bufs, t, demand=D)
        torch.cuda.synchronize()
        h = {k: getattr(out, k).cpu().numpy() for k in (
            "t_balance", "t_intra", "scale_out", "redistribution", "total", "t_optimal",
            "t_worstcase", "assumption_ok", "so_weight", "so_server", "so_demand", "so_total",
            "status")}
        n_stages = bufs.n_stages.cpu().numpy()
        for b, r in enumerate(rows):
            assert int(h["status"][b]) == 0, r["name"]
            _check_fields({k: v[b] for k, v in h.items()}, r, int(n_stages[b]))


@pytest.mark.gpu
def test_object_api_matches_reference():
    """simulate_fast(plan, stages, t) / simulate_spreadout / bounds / spreadout
    stages through the drop-in object API (device kernel underneath)."""
    import warnings

    import paper_2505_09764_b200 as fb

    for r in _golden()[::3]:
        n, m = r["n"], r["m"]
        b1, b2, a = (_f(x) for x in r["topo"])
        t = fb.Topology(n, m, scaleup_bw=b1, scaleout_bw=b2, wakeup_delay=a)
        d = fb.DemandMatrix(n, m, np.array(r["sizes"], np.int64))
        sched = fb.synthesize_fast(d, t)
        line = fb.simulate_fast(sched.plan, list(sched.stages), t)
        want = r["fast"]
        assert float(line.t_balance).hex() == want["t_balance"], r["name"]
        assert float(line.t_intra_a2a).hex() == want["t_intra_a2a"], r["name"]
        assert _hex(line.scale_out) == want["scale_out"], r["name"]
        assert _hex(line.redistribution) == want["redistribution"], r["name"]
        assert float(line.total).hex() == want["total"], r["name"]
        server = fb.reduce_to_server_level(d, t)
        so = fb.simulate_spreadout(server, t)
        assert _hex(so.scale_out) == r["spreadout"]["scale_out"]
        assert float(so.total).hex() == r["spreadout"]["total"]
        sod = fb.simulate_spreadout(server, t, demand=d)
        assert _hex(sod.scale_out) == r["spreadout_demand"]["scale_out"]
        assert float(sod.total).hex() == r["spreadout_demand"]["total"]
        assert [s.weight for s in fb.spreadout_stages(server)] == r["spreadout_weights"]
        assert fb.spreadout_completion_units(server) == r["spreadout_units"]
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            assert float(fb.optimal_time(server, t)).hex() == r["t_optimal"]
            assert float(fb.fast_worstcase_time(server, t)).hex() == r["t_worstcase"]
        assert float(fb.ratio_bound(t)).hex() == r["ratio_bound"]
        assert fb.intra_assumption_holds(server) == r["assumption_ok"]


@pytest.mark.gpu
def test_model_structure_cases():
    """The reference's structural tests (test_simulate.py:47-122, 197-225)."""
    import paper_2505_09764_b200 as fb

    t = fb.Topology(3, 2, scaleup_bw=4 * 50e9, scaleout_bw=50e9)
    d = fb.gen_zipf(0, t, 0.8, 100_000)
    sched = fb.synthesize_fast(d, t)
    stages = list(sched.stages)
    assert len(stages) >= 2 and stages[0].weight < stages[-1].weight
    with pytest.raises(fb.ValidationError, match="ascending"):
        fb.simulate_fast(sched.plan, stages[::-1], t)
    # zero demand costs nothing
    t2 = fb.Topology(2, 2, scaleup_bw=4 * 50e9, scaleout_bw=50e9)
    z = fb.DemandMatrix(2, 2, np.zeros((4, 4), dtype=np.int64))
    sz = fb.synthesize_fast(z, t2)
    line = fb.simulate_fast(sz.plan, list(sz.stages), t2)
    assert line.total == 0.0 and line.scale_out == ()
    # intra-only demand: one scale-up phase
    t3 = fb.Topology(2, 2, scaleup_bw=4 * 50e9, scaleout_bw=50e9, wakeup_delay=0.25)
    sizes = np.zeros((4, 4), dtype=np.int64)
    sizes[0, 1] = 100 * 10**9
    si = fb.synthesize_fast(fb.DemandMatrix(2, 2, sizes), t3)
    line = fb.simulate_fast(si.plan, list(si.stages), t3)
    assert line.scale_out == () and line.total == pytest.approx(0.25 + 100e9 / t3.scaleup_bw)
    # stage bytes must match the tables
    sizes = np.zeros((4, 4), dtype=np.int64)
    sizes[0, 2] = 10
    st = fb.synthesize_fast(fb.DemandMatrix(2, 2, sizes), t2)
    tampered = [fb.PermutationStage(weight=s.weight, edges=tuple((a, b, x - 1) for a, b, x in s.edges))
                for s in st.stages]
    with pytest.raises(fb.InternalInvariantError):
        fb.simulate_fast(st.plan, tampered, t2)
    # hand-checked pipeline arithmetic
    tk = fb.Topology(2, 1, scaleup_bw=100.0, scaleout_bw=10.0, wakeup_delay=0.5)
    sk = fb.synthesize_fast(fb.DemandMatrix(2, 1, np.array([[0, 40], [60, 0]], np.int64)), tk)
    line = fb.simulate_fast(sk.plan, list(sk.stages), tk)
    assert line.t_balance == 0.0 and line.t_intra_a2a == 0.0
    assert line.scale_out == (0.5 + 60 / 10.0,) and line.total == pytest.approx(6.5)
    # spreadout: server-level hand arithmetic, raw mode charging GPU imbalance
    ts3 = fb.Topology(3, 2, scaleup_bw=100.0, scaleout_bw=10.0, wakeup_delay=1.0)
    s = fb.ServerMatrix(totals=np.array([[0, 40, 0], [0, 0, 20], [60, 0, 0]], np.int64))
    so = fb.simulate_spreadout(s, ts3)
    assert so.scale_out == (1.0 + 30 / 10.0, 0.0) and so.total == pytest.approx(4.0)
    sizes = np.zeros((4, 4), dtype=np.int64)
    sizes[0, 2] = 1000
    dd = fb.DemandMatrix(2, 2, sizes)
    ss = fb.reduce_to_server_level(dd, t2)
    assert fb.simulate_spreadout(ss, t2, demand=dd).total == pytest.approx(
        2 * fb.simulate_spreadout(ss, t2).total)
    with pytest.raises(fb.ValidationError):
        fb.simulate_spreadout(fb.ServerMatrix(totals=np.zeros((2, 2), np.int64)), t)
    # move-list equivalence (test_simulate.py:169-192)
    t4 = fb.Topology(3, 4, scaleup_bw=8 * 50e9, scaleout_bw=50e9)
    d4 = fb.gen_zipf(3, t4, 0.8, 1_000_000_000)
    s4 = fb.synthesize_fast(d4, t4)
    line = fb.simulate_fast(s4.plan, list(s4.stages), t4)
    earlier: dict = {}
    for k, stage in enumerate(s4.stages):
        moves = fb.stage_redistribution(s4.plan, [(a, b) for a, b, _ in stage.edges],
                                        delivered={(a, b): x for a, b, x in stage.edges},
                                        earlier={p: list(v) for p, v in earlier.items()})
        assert fb.intra_phase_time(moves, t4) == pytest.approx(line.redistribution[k], rel=1e-12,
                                                               abs=1e-18)
        for a, b, x in stage.edges:
            earlier.setdefault((a, b), []).append(x)
