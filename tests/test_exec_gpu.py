"""Executor parity on one B200 (group mode): every rank's receive buffer is
byte-identical to the direct-alltoallv oracle.

GroupComm puts all ranks' symmetric blocks on one device and runs the SAME
exec kernel for all ranks in one cooperative launch, so the full protocol
(entry barrier, per-phase counters, staging, redistribution, epochs) is
exercised without multi-process kernels that wait on each other.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle
from oracle.alltoallv import direct_alltoallv, payload
from paper_2505_09764_b200 import Topology, workloads
from paper_2505_09764_b200.executor import OP_DTYPE, GroupComm, plan_compile_host
from paper_2505_09764_b200.schedule import PackedSchedule

pytestmark = pytest.mark.gpu


def _sends(D):
    return [torch.from_numpy(payload(g, int(D[g].sum()) + 16)).cuda() for g in range(D.shape[0])]


def _check(comm: GroupComm, D: np.ndarray, sends_np=None):
    G = D.shape[0]
    sends_np = sends_np or [payload(g, int(D[g].sum()) + 16) for g in range(G)]
    sends = [torch.from_numpy(s).cuda() for s in sends_np]
    recvs = comm.alltoallv(sends, torch.from_numpy(D).cuda())
    torch.cuda.synchronize()
    comm.check()
    want = direct_alltoallv(sends_np, D)
    for h in range(G):
        got = recvs[h][: len(want[h])].cpu().numpy()
        assert np.array_equal(got, want[h]), f"rank {h}"
    return comm


def _comm_for(n, m, D, blocks=8, chunk=64 * 1024):
    cap = int(max(D.sum(axis=0).max(), D.sum(axis=1).max())) + 4096
    return GroupComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20),
                     blocks=blocks, chunk_bytes=chunk)


@pytest.mark.parametrize("n,m", [(2, 1), (2, 2), (4, 1), (2, 4), (4, 2), (8, 1), (3, 2)])
def test_group_exec_matches_direct_alltoallv(n, m):
    G = n * m
    rng = np.random.default_rng(100 + G * 10 + m)
    cases = [workloads.zipf_sizes(1, G, 1.2, 3_000_017),
             workloads.gen_uniform(2, Topology(n, m), 77_777).sizes,
             workloads.gen_adversarial(Topology(n, m), 123_457).sizes]
    D = rng.integers(0, 300_000, (G, G)).astype(np.int64)
    D[rng.random((G, G)) < 0.5] = 0
    np.fill_diagonal(D, 0)
    cases.append(D)
    cap = max(int(max(c.sum(0).max(), c.sum(1).max())) for c in cases) + 4096
    comm = GroupComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20),
                     blocks=8, chunk_bytes=64 * 1024)
    for D in cases:  # several epochs on one communicator
        _check(comm, D)
    comm.close()


def test_group_exec_config2_scale():
    # BASELINE config 2 instance: Zipf 1.2, 256 MiB total, 2 x 4 virtual servers
    D = workloads.zipf_sizes(0, 8, 1.2, 268_435_456)
    comm = _comm_for(2, 4, D, blocks=16, chunk=256 * 1024)
    _check(comm, D)
    _check(comm, D)
    comm.close()


def test_device_plan_equals_host_plan():
    n, m = 4, 2
    D = workloads.zipf_sizes(3, 8, 0.9, 5_000_011)
    comm = _comm_for(n, m, D)
    _check(comm, D)
    dev_ops = comm.plan.host_ops()
    out = oracle.synthesize_batch(D, n, m)
    p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
    host_ops, used, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm, p.stage_bytes,
                                           comm.recv_bytes, comm.staging_bytes, chunk=comm.chunk)
    assert st == 0
    assert dev_ops.dtype == OP_DTYPE
    assert np.array_equal(dev_ops, host_ops)
    assert np.array_equal(comm.plan.staging_used.cpu().numpy(), used)
    comm.close()


def _device_plan(D, n, m, selfb, recv_cap, staging_cap, chunk):
    """fast_synth_batch + fast_plan_compile (CTA-parallel build) on cuda:0."""
    import ctypes

    from paper_2505_09764_b200 import _lib, synth
    from paper_2505_09764_b200.executor import PlanBuffers

    lib = _lib.load()
    Dd = torch.from_numpy(D).cuda().view(1, n * m, n * m)
    sd = torch.from_numpy(selfb).cuda()
    bufs = synth.SynthBuffers(1, n, m)
    plan = PlanBuffers(n, m, "cuda")
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.fast_synth_batch(ctypes.c_void_p(Dd.data_ptr()), 1, n, m,
                                ctypes.byref(bufs.struct), sh) == 0
    assert lib.fast_plan_compile(ctypes.c_void_p(Dd.data_ptr()), ctypes.c_void_p(sd.data_ptr()),
                                 n, m, ctypes.byref(bufs.struct), recv_cap, staging_cap, chunk,
                                 ctypes.byref(plan.struct), sh) == 0
    torch.cuda.synchronize()
    return plan.host_ops(), plan.staging_used.cpu().numpy(), int(plan.status.item())


@pytest.mark.parametrize("n,m", [(2, 1), (2, 2), (2, 4), (4, 2), (3, 3), (8, 1), (2, 8),
                                 (4, 4), (5, 2), (6, 3), (3, 8)])
def test_parallel_device_plan_equals_host_plan(n, m):
    """The CTA-parallel device plan (plan_par.cuh) is op-for-op identical to
    the sequential host build (plan.cuh) -- Zipf, sparse, uniform and
    hotspot matrices, power-of-two and odd chunk sizes, with self segments."""
    G = n * m
    rng = np.random.default_rng(7 * G + m)
    sparse = rng.integers(1, 900_000, (G, G)).astype(np.int64)
    sparse[rng.random((G, G)) < 0.6] = 0
    np.fill_diagonal(sparse, 0)
    cases = [workloads.zipf_sizes(5, G, 1.2, 40_000_003), sparse,
             workloads.gen_uniform(3, Topology(n, m), 65_537).sizes,
             workloads.gen_hotspot(4, Topology(n, m), 3_000_001, G - 1, 8).sizes,
             np.ones((G, G), np.int64) - np.eye(G, dtype=np.int64)]
    for ci, D in enumerate(cases):
        D = np.ascontiguousarray(D, dtype=np.int64)
        selfb = rng.integers(0, 5000, G).astype(np.int64) if ci % 2 else np.zeros(G, np.int64)
        out = oracle.synthesize_batch(D, n, m)
        p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
        cap = int((D.sum(axis=0) + selfb).max()) + 64
        stg = 4 * cap + (1 << 20)
        for chunk in (64 * 1024, 1 << 20, 48 * 1024 + 16):
            host_ops, used, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm,
                                                   p.stage_bytes, cap, stg, send_self=selfb,
                                                   chunk=chunk)
            dev_ops, dused, dst = _device_plan(D, n, m, selfb, cap, stg, chunk)
            assert st == 0 and dst == 0, (ci, chunk, st, dst)
            assert dev_ops.dtype == OP_DTYPE
            assert np.array_equal(dev_ops, host_ops), (ci, chunk, len(dev_ops), len(host_ops))
            assert np.array_equal(dused, used), (ci, chunk)
    # too-small receive / staging buffers: same status as the host build
    D = np.ascontiguousarray(cases[0], dtype=np.int64)
    out = oracle.synthesize_batch(D, n, m)
    p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
    z = np.zeros(G, np.int64)
    for rc, sc in [(16, 1 << 40), (1 << 40, 16)]:
        _, _, st = plan_compile_host(D, n, m, p.stage_order, p.stage_perm, p.stage_bytes, rc, sc,
                                     send_self=z, chunk=1 << 20)
        _, _, dst = _device_plan(D, n, m, z, rc, sc, 1 << 20)
        assert st == dst, (rc, sc, st, dst)
        assert rc > 16 or st != 0


def test_group_exec_reports_small_buffers():
    n, m = 2, 2
    D = workloads.zipf_sizes(1, 4, 0.5, 100_000)
    comm = GroupComm(Topology(n, m), recv_bytes=1000, staging_bytes=1000)
    sends = _sends(D)
    comm.alltoallv(sends, torch.from_numpy(D).cuda())
    torch.cuda.synchronize()
    from paper_2505_09764_b200 import ValidationError

    with pytest.raises(ValidationError):
        comm.check()
    comm.close()


def test_group_exec_edge_cases():
    """Empty traffic, 1-byte and sub-16-byte (misaligned) segments, a single
    huge segment, and changing traffic across epochs on one communicator."""
    n, m = 2, 4
    G = n * m
    rng = np.random.default_rng(5)
    cases = [np.zeros((G, G), np.int64)]
    one = np.zeros((G, G), np.int64)
    one[3, 6] = 1
    cases.append(one)
    tiny = rng.integers(0, 16, (G, G)).astype(np.int64)
    np.fill_diagonal(tiny, 0)
    cases.append(tiny)
    huge = np.zeros((G, G), np.int64)
    huge[0, 7] = 50_000_017
    cases.append(huge)
    odd = rng.integers(1, 70_000, (G, G)).astype(np.int64) * 3 + 1
    np.fill_diagonal(odd, 0)
    cases.append(odd)
    cap = max(int(max(c.sum(0).max(), c.sum(1).max())) for c in cases) + 4096
    comm = GroupComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20),
                     blocks=8, chunk_bytes=64 * 1024)
    for D in cases + cases[::-1]:
        _check(comm, D)
    comm.close()


@pytest.mark.parametrize("n,m", [(8, 1), (2, 8)])
def test_group_exec_wide_partitions(n, m):
    G = n * m
    D = workloads.zipf_sizes(7, G, 1.1, 20_000_003)
    cap = int(max(D.sum(0).max(), D.sum(1).max())) + 4096
    comm = GroupComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20),
                     blocks=max(1, 144 // G), chunk_bytes=64 * 1024)
    _check(comm, D)
    _check(comm, workloads.gen_adversarial(Topology(n, m), 1_000_003).sizes)
    comm.close()


@pytest.mark.parametrize("n,m", [(2, 4), (4, 2)])
def test_group_exec_measured_timeline(n, m):
    """The measured Timeline (the reference's phase breakdown,
    simulate.py:38-55) is filled from device stamps: every phase that has
    chunks has a non-empty window, windows lie inside [0, total], the stage
    sends follow the plan's phase order (balance before the stages that
    forward balanced-in bytes), and the slowest rank's total matches the CUDA
    event time of the exec kernel within 5 %."""
    from paper_2505_09764_b200.executor import PH_BALANCE, PH_REDIST, STAGE_INTRA

    D = workloads.zipf_sizes(0, n * m, 1.2, 1 << 28)
    comm = _comm_for(n, m, D, blocks=16, chunk=1 << 20)
    sends = _sends(D)
    Dt = torch.from_numpy(D).cuda()
    comm.alltoallv(sends, Dt)  # warm-up
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    comm.alltoallv(sends, Dt, exec_events=ev)
    torch.cuda.synchronize()
    comm.check()
    ops = comm.plan.host_ops()
    totals = []
    for r in range(n * m):
        tl = comm.measured_timeline(r)
        ph = comm.measured_phases(r)
        mine = ops[ops["exec_rank"] == r]
        assert tl.total > 0 and ph["barrier"] >= 0
        has_bal = bool((mine["phase"] == PH_BALANCE).any())
        has_intra = bool((mine["stage"] == STAGE_INTRA).any())
        assert (tl.t_balance > 0) == has_bal and (tl.t_intra_a2a > 0) == has_intra, r
        for k in range(len(tl.scale_out)):
            sel = mine[mine["stage"] == k]
            assert (tl.scale_out[k] > 0) == bool((sel["phase"] != PH_REDIST).any()), (r, k)
            assert (tl.redistribution[k] > 0) == bool((sel["phase"] == PH_REDIST).any()), (r, k)
        wins = [w for w in [ph["balance"], ph["intra"], *ph["scale_out"], *ph["redistribution"]]
                if w is not None]
        for a, b in wins:
            assert ph["barrier"] <= a <= b <= tl.total + 1e-6, (r, a, b, tl.total)
        totals.append(tl.total)
    ev_s = ev[0].elapsed_time(ev[1]) * 1e-3
    assert abs(max(totals) - ev_s) <= 0.05 * ev_s, (max(totals), ev_s)
    comm.close()


@pytest.mark.parametrize("n,m", [(2, 2), (2, 4), (4, 2)])
def test_group_exec_copy_self(n, m):
    """FAST_PLAN_COPY_SELF: the exec CTAs also move each rank's own segment
    (kept in place in its send buffer) into the gap at its receive slot, so
    every receive buffer is the complete all_to_all_single output."""
    G = n * m
    D = workloads.zipf_sizes(7, G, 1.2, 2_000_003)
    selfb = np.array([12_345 + 1_001 * g for g in range(G)], dtype=np.int64)
    Dfull = D + np.diag(selfb)
    cap = int(Dfull.sum(axis=0).max()) + 4096
    comm = GroupComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20), blocks=8,
                     chunk_bytes=64 * 1024)
    sends_np = [payload(g, int(Dfull[g].sum()) + 16) for g in range(G)]
    recvs = comm.alltoallv([torch.from_numpy(x).cuda() for x in sends_np],
                           torch.from_numpy(D).cuda(), self_bytes=torch.from_numpy(selfb).cuda(),
                           copy_self=True)
    torch.cuda.synchronize()
    comm.check()
    want = direct_alltoallv(sends_np, Dfull)
    for h in range(G):
        assert np.array_equal(recvs[h][: len(want[h])].cpu().numpy(), want[h]), h
    comm.close()
