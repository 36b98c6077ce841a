"""Executor plan (Appendix-A byte placement) validated on the CPU.

The host build of plan.cuh (fast_plan_compile_host -- the same code the
device runs as a one-thread kernel) turns an oracle schedule into copy ops;
replaying them on numpy buffers must reproduce a direct alltoallv byte for
byte, and the ops must realise exactly the reference schedule: per GPU pair
the balance bytes equal the schedule's IntraMoves, stage sends go from lane
p to the same-index proxy, and each stage moves exactly its edge bytes.
"""

from __future__ import annotations

from collections import defaultdict

import numpy as np
import pytest

from oracle import oracle
from oracle.alltoallv import direct_alltoallv, payload
from paper_2505_09764_b200 import workloads
from paper_2505_09764_b200.executor import (BUF_RECV, BUF_SEND, BUF_STAGING, PH_BALANCE,
                                            PH_DIRECT, PH_FROM_STAGING, PH_REDIST,
                                            plan_compile_host)
from paper_2505_09764_b200.schedule import PackedSchedule


def replay(ops, sends, G, recv_cap, stg_cap):
    recv = [np.zeros(recv_cap, np.uint8) for _ in range(G)]
    stg = [np.zeros(stg_cap + 64, np.uint8) for _ in range(G)]
    for o in ops:
        e, d = int(o["exec_rank"]), int(o["dst_rank"])
        so, do, ln = int(o["src_off"]), int(o["dst_off"]), int(o["len"])
        src = sends[e] if o["src_buf"] == BUF_SEND else stg[e]
        dst = recv[d] if o["dst_buf"] == BUF_RECV else stg[d]
        assert len(src[so:so + ln]) == ln and len(dst[do:do + ln]) == ln
        dst[do:do + ln] = src[so:so + ln]
    return recv


def check_flags(ops, chunk):
    """Every staging consumer waits on exactly the producer chunks that write
    its source bytes (the executor's per-chunk flag protocol)."""
    producers = {}
    for o in ops:
        if o["sig_slot"] >= 0:
            assert o["dst_buf"] == BUF_STAGING
            producers[(int(o["dst_rank"]), int(o["sig_slot"]))] = o
        else:
            assert o["dst_buf"] == BUF_RECV
    slots = defaultdict(set)
    for (r, s0), o in producers.items():
        nch = (int(o["len"]) + chunk - 1) // chunk
        for c in range(nch):
            assert (s0 + c) not in slots[r], "flag slots overlap"
            slots[r].add(s0 + c)
    for o in ops:
        if o["src_buf"] == BUF_STAGING:
            assert o["wait_slot"] >= 0
            prod = producers[(int(o["exec_rank"]), int(o["wait_slot"]))]
            lo = int(prod["dst_off"]) + int(o["wait_off"])
            assert int(o["src_off"]) == lo
            assert int(o["wait_off"]) + int(o["len"]) <= int(prod["len"])
        else:
            assert o["wait_slot"] < 0


def check_instance(D: np.ndarray, n: int, m: int, chunk: int = 4096):
    G = n * m
    out = oracle.synthesize_batch(D, n, m)
    assert int(out["status"][0]) == 0
    p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
    recv_cap = int(D.sum(axis=0).max()) + 16
    stg_cap = int(D.sum()) + 16 * G * G * 4 + 1024
    ops, used, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm, p.stage_bytes,
                                      recv_cap, stg_cap, chunk=chunk)
    assert st == 0
    check_flags(ops, chunk)
    assert (used <= stg_cap).all()
    # phase order
    assert np.all(np.diff(ops["phase"].astype(int)) >= 0)
    assert (ops["len"] > 0).all()
    sends = [payload(g, int(D[g].sum())) for g in range(G)]
    got = replay(ops, sends, G, recv_cap, stg_cap)
    want = direct_alltoallv(sends, D)
    for h in range(G):
        assert np.array_equal(got[h][:len(want[h])], want[h]), h
    # balance ops realise the schedule's IntraMoves per (server, from, to)
    mv = defaultdict(int)
    for (srv, f, t, _dst, b) in p.move_list():
        mv[(srv * m + f, srv * m + t)] += b
    bal = defaultdict(int)
    for o in ops[ops["phase"] == PH_BALANCE]:
        assert o["src_buf"] == BUF_SEND and o["dst_buf"] == BUF_STAGING
        bal[(int(o["exec_rank"]), int(o["dst_rank"]))] += int(o["len"])
    assert dict(bal) == dict(mv)
    # stage sends: lane p -> proxy p of the destination server; bytes per
    # (stage, src server, dst server) equal the sorted stage's edge bytes
    per_stage = defaultdict(int)
    sends_ops = ops[(ops["phase"] == PH_DIRECT) | (ops["phase"] == PH_FROM_STAGING)]
    for o in sends_ops:
        e, d = int(o["exec_rank"]), int(o["dst_rank"])
        if e // m == d // m:
            assert o["phase"] == PH_DIRECT and o["dst_buf"] == BUF_RECV  # intra tile
            assert o["stage"] == 255  # FAST_STAGE_INTRA
            continue
        assert e % m == d % m, "stage traffic must go lane p -> proxy p"
        per_stage[(int(o["stage"]), e // m, d // m)] += int(o["len"])
    want_stage = {}
    for s_idx, k in enumerate(p.stage_order):
        for u in range(n):
            b = int(p.stage_bytes[k][u])
            if b > 0:
                want_stage[(s_idx, u, int(p.stage_perm[k][u]))] = b
    assert dict(per_stage) == want_stage
    # redistribution stays inside the destination server, proxy -> final GPU
    for o in ops[ops["phase"] == PH_REDIST]:
        e, d = int(o["exec_rank"]), int(o["dst_rank"])
        assert e // m == d // m and e != d and o["src_buf"] == BUF_STAGING
    return ops


@pytest.mark.parametrize("n,m", [(2, 1), (2, 2), (2, 4), (4, 2), (3, 3), (4, 1), (8, 1),
                                 (2, 8), (3, 2), (5, 3)])
def test_plan_replays_to_direct_alltoallv(n, m):
    G = n * m
    rng = np.random.default_rng(7 * n + m)
    for trial in range(12):
        if trial % 4 == 0:
            D = workloads.zipf_sizes(trial, G, 1.2, int(rng.integers(1000, 200_000)))
        elif trial % 4 == 1:
            D = workloads.gen_uniform(trial, workloads.Topology(n, m), 3000).sizes
        elif trial % 4 == 2:
            D = rng.integers(0, 5000, (G, G)).astype(np.int64)
            D[rng.random((G, G)) < 0.6] = 0
            np.fill_diagonal(D, 0)
        else:
            D = workloads.gen_adversarial(workloads.Topology(n, m), 777 + trial).sizes
        check_instance(D, n, m)


def test_plan_baseline_configs():
    # seed-0 instances of BASELINE configs 1/2 shapes, scaled down 1/1024
    for n, m in [(2, 4), (4, 2)]:
        check_instance(workloads.zipf_sizes(0, 8, 1.2, 268_435_456 // 1024), n, m)
        check_instance(workloads.zipf_sizes(0, 8, 0.0, 67_108_864 // 1024), n, m)


def test_plan_rejects_small_buffers():
    n, m = 2, 2
    D = workloads.zipf_sizes(1, 4, 0.5, 10_000)
    out = oracle.synthesize_batch(D, n, m)
    p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
    _, _, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm, p.stage_bytes,
                                 int(D.sum(axis=0).max()) - 1, 1 << 20)
    assert st == 2
    _, _, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm, p.stage_bytes,
                                 1 << 20, 0)
    assert st == 2


def test_plan_self_segments_stay_in_place():
    """all_to_all_single layout: send_g keeps its own segment in place."""
    rng = np.random.default_rng(3)
    for n, m in [(2, 1), (2, 4), (4, 2)]:
        G = n * m
        D = workloads.zipf_sizes(9, G, 1.1, 400_009)
        selfb = rng.integers(0, 5000, G).astype(np.int64)
        out = oracle.synthesize_batch(D, n, m)
        p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
        cap = int((D + np.diag(selfb)).sum(axis=0).max()) + 16
        stg = int(D.sum()) + 1 << 16
        ops, _, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm, p.stage_bytes,
                                       cap, stg, send_self=selfb)
        assert st == 0
        Dfull = D + np.diag(selfb)
        sends = [payload(g, int(Dfull[g].sum())) for g in range(G)]
        got = replay(ops, sends, G, cap, stg)
        full = direct_alltoallv(sends, Dfull)
        for h in range(G):
            lo = int(Dfull[:h, h].sum())
            # the self slot is a gap; everything else is all_to_all_single's output
            assert np.array_equal(got[h][:lo], full[h][:lo]), (n, m, h)
            hi = lo + int(selfb[h])
            assert np.array_equal(got[h][hi:len(full[h])], full[h][hi:]), (n, m, h)
