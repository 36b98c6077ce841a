"""alltoallv benchmark for bench.py at N > 1 (torchrun, one rank per GPU).

Workload (BASELINE config 2 shape): Zipf alpha=1.2 traffic matrix with a
256 MiB total over the N GPUs, virtual servers 2 x N/2 (N=8: 2x4; --topo
4x2 for the other partition).  One step = one FastComm.alltoallv: P2P
demand all-gather + FAST synthesis + plan compile + P2P stage execution,
all on the device.  Timed with CUDA events, max over ranks.
"""

from __future__ import annotations

import json
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from bench import ClockSampler, measured_peaks

PEER_GBS = 770.0      # measured B200 peer copy per direction (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0


def topology_for(world: int, spec: str | None):
    if spec:
        n, m = (int(x) for x in spec.lower().split("x"))
        return n, m
    return (2, world // 2) if world >= 2 else (1, 1)


def demand(args, world: int) -> np.ndarray:
    from paper_2505_09764_b200 import workloads

    return workloads.zipf_sizes(args.seed, world, args.a2a_skew, args.a2a_total)


class NvlinkCounters:
    """NVML NVLink data throughput counters (KiB, cumulative, summed over the
    GPU's links) for the GPU behind a CUDA device index -- ncu cannot replay
    the exec kernel (its ranks wait on each other), NVML counts the wire
    traffic of the real multi-rank run."""

    FIELD_TX, FIELD_RX = 138, 139  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX

    def __init__(self, device_index: int):
        self.h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            p = torch.cuda.get_device_properties(device_index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.links = [l for l in range(18)
                          if self._state(l)]
        except Exception:  # pragma: no cover - NVML absent
            self.h = None

    def _state(self, link: int) -> bool:
        try:
            return self.nv.nvmlDeviceGetNvLinkState(self.h, link) == 1
        except Exception:
            return False

    def read(self):
        """(tx_bytes, rx_bytes) or None."""
        if self.h is None or not self.links:
            return None
        try:
            ids = [(self.FIELD_TX, l) for l in self.links] + [(self.FIELD_RX, l) for l in self.links]
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, ids)
            tot = [0, 0]
            for i, v in enumerate(vals):
                if v.nvmlReturn != 0:
                    return None
                tot[0 if i < len(self.links) else 1] += int(v.value.ullVal)
            return tot[0] * 1024, tot[1] * 1024
        except Exception:
            return None


def peer_copy_peaks(comm, rank: int, nbytes: int) -> dict | None:
    """In-run NVLink push peaks, rank 0 -> rank 1's receive region: the
    executor's SM copy loop (fast_debug_copy, 128 CTAs) and the copy engine
    (cudaMemcpyAsync); GB/s per direction, best of 5 (other ranks idle)."""
    import ctypes

    from paper_2505_09764_b200 import _lib

    lib = _lib.load()
    res = None
    dist.barrier()
    if rank == 0:
        dst = lib.fast_comm_peer_ptr(comm._ptr, 1)
        recv_off = lib.fast_comm_recv_ptr(comm._ptr) - lib.fast_comm_peer_ptr(comm._ptr, 0)
        src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream()
        out = {}
        for name in ("sm_copy", "copy_engine"):
            best = 1e9
            for _ in range(6):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                if name == "sm_copy":
                    lib.fast_debug_copy(ctypes.c_void_p(dst + recv_off),
                                        ctypes.c_void_p(src.data_ptr()), nbytes, 128, 1 << 20, 1,
                                        ctypes.c_void_p(s.cuda_stream))
                else:
                    lib.fast_debug_memcpy(ctypes.c_void_p(dst + recv_off),
                                          ctypes.c_void_p(src.data_ptr()), nbytes,
                                          ctypes.c_void_p(s.cuda_stream))
                b.record(s)
                b.synchronize()
                best = min(best, a.elapsed_time(b))
            out[name] = round(nbytes / (best * 1e-3) / 1e9, 1)
        res = {"bytes": nbytes, "GBps": out, "what": "push rank0 -> rank1, best of 5"}
    torch.cuda.synchronize()
    dist.barrier()
    return res


def timeline_vs_model(D: np.ndarray, n: int, m: int, tls: list, peaks_run) -> dict:
    """Measured Timeline (rank 0 and the slowest rank; seconds) beside
    simulate_fast's model of the same schedule (simulate.py:107-193) with both
    tiers at the in-run SM-store peer peak (one NVLink tier)."""
    from paper_2505_09764_b200 import DemandMatrix, Topology, simulate_fast, synthesize_fast

    bw = (peaks_run["GBps"]["sm_copy"] if peaks_run else PEER_GBS) * 1e9
    t = Topology(n, m, bw, bw)
    sch = synthesize_fast(DemandMatrix(n, m, np.asarray(D, np.int64)), t)
    model = simulate_fast(sch.plan, list(sch.stages), t).to_json_dict()
    slow = max(range(len(tls)), key=lambda r: tls[r]["total"])
    r6 = lambda d: {k: (round(v * 1e6, 2) if isinstance(v, float) else  # noqa: E731
                        [round(x * 1e6, 2) for x in v]) for k, v in d.items()}
    return {"unit": "us", "measured_rank0": r6(tls[0]), "measured_slowest_rank": slow,
            "measured_slowest": r6(tls[slow]), "model_simulate_fast": r6(model),
            "model_bandwidth_GBps": round(bw / 1e9, 1),
            "note": "measured: device %globaltimer windows of one call (phase durations; total = "
                    "exec start to the rank's last send and arrival); model: the reference's "
                    "pipelined cost model, both tiers at the measured SM-store peer peak"}


def fast_wire_bytes(ops: np.ndarray, G: int) -> tuple[int, int]:
    eg = np.zeros(G, np.int64)
    ing = np.zeros(G, np.int64)
    for o in ops:
        if int(o["exec_rank"]) != int(o["dst_rank"]):
            eg[int(o["exec_rank"])] += int(o["len"])
            ing[int(o["dst_rank"])] += int(o["len"])
    return int(eg.max()), int(ing.max())


# NCCL knobs of the comparison bar: all_to_all_single on this traffic runs
# 1.5-1.9x faster with 64 P2P channels than with the defaults
# (profiles/r2_nccl_sweep_n*.log), so the bar uses them (overridable).
NCCL_TUNED = {"NCCL_NCHANNELS_PER_PEER": "32", "NCCL_MIN_P2P_NCHANNELS": "64",
              "NCCL_MAX_P2P_NCHANNELS": "64"}


def _tune_nccl() -> dict:
    if os.environ.get("FAST_BENCH_NCCL_DEFAULTS") != "1":
        for k, v in NCCL_TUNED.items():
            os.environ.setdefault(k, v)
    return {k: os.environ[k] for k in NCCL_KNOBS if k in os.environ}


def run(args, workload: str) -> dict | None:
    nccl_env = _tune_nccl()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return reference_alltoallv(args, world) if rank == 0 else None
    if world < 2:
        return {"metric": "alltoallv algbw", "unavailable": "alltoallv needs >= 2 ranks (torchrun)"}
    from paper_2505_09764_b200 import Topology, algorithmic_bandwidth
    from paper_2505_09764_b200.executor import FastComm

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, m = topology_for(world, args.topo)
    D = demand(args, world)
    G = world
    if getattr(args, "nccl_only", False):
        return nccl_only(args, D, rank, world)
    total = int(D.sum())
    cap = int(max(D.sum(0).max(), D.sum(1).max())) + 4096
    comm = FastComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (4 << 20),
                    blocks=args.blocks, chunk_bytes=args.chunk)
    row = torch.from_numpy(D[rank].copy()).cuda()
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    send = torch.randint(0, 256, (int(D[rank].sum()) + 16,), dtype=torch.uint8, device="cuda",
                         generator=gen)
    stream = torch.cuda.current_stream()

    # correctness vs NCCL on the same bytes (not timed)
    recv = comm.alltoallv(send, row)
    nccl_out = torch.empty(int(D[:, rank].sum()), dtype=torch.uint8, device="cuda")
    dist.all_to_all_single(nccl_out, send[: int(D[rank].sum())], D[:, rank].tolist(),
                           D[rank].tolist())
    torch.cuda.synchronize()
    comm.check()
    ok = torch.equal(recv[: nccl_out.numel()], nccl_out)
    okt = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(okt)
    if int(okt.item()) != 0:
        raise RuntimeError("FAST alltoallv result differs from NCCL all_to_all_single")

    # timed: the product call (CUDA-graph replay of gather+synthesis+plan+exec)
    for _ in range(args.warmup):
        comm.alltoallv(send, row)
    torch.cuda.synchronize()
    dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            comm.alltoallv(send, row)
        t1.record(stream)
        torch.cuda.synchronize()
    comm.check()
    step_ms = t0.elapsed_time(t1) / args.steps
    # exec kernel alone (same traffic, step-by-step path with events around it),
    # with the NVML NVLink data counters read around the loop
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    nvl = NvlinkCounters(local)
    torch.cuda.synchronize()
    dist.barrier()
    c0 = nvl.read()
    for k in range(args.steps):
        comm.alltoallv(send, row, exec_events=ev[k])
    torch.cuda.synchronize()
    c1 = nvl.read()
    dist.barrier()
    comm.check()
    exec_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    my_exec_ms = exec_ms
    mx = torch.tensor([step_ms, exec_ms], device="cuda")
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    step_ms, exec_ms = (float(x) for x in mx.tolist())
    nvl_rank = None
    if c0 is not None and c1 is not None:
        tx, rx = (c1[0] - c0[0]) / args.steps, (c1[1] - c0[1]) / args.steps
        nvl_rank = [tx, rx, my_exec_ms]
    nvl_all = [None] * world
    dist.all_gather_object(nvl_all, nvl_rank)
    peaks_run = peer_copy_peaks(comm, rank, min(comm.recv_bytes - 4096, 128 << 20))
    # measured per-phase Timeline of one call (device %globaltimer windows),
    # every rank, next to the reference's analytical model of the same schedule
    comm.alltoallv(send, row, record_timeline=True)
    torch.cuda.synchronize()
    comm.check()
    tl = comm.measured_timeline()
    tls = [None] * world
    dist.all_gather_object(tls, tl.to_json_dict())

    # NCCL all_to_all_single on the identical traffic (practical B200 bar)
    ins, outs = D[rank].tolist(), D[:, rank].tolist()
    sv = send[: int(D[rank].sum())]
    for _ in range(args.warmup):
        dist.all_to_all_single(nccl_out, sv, outs, ins)
    torch.cuda.synchronize()
    dist.barrier()
    n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0.record(stream)
    for _ in range(args.steps):
        dist.all_to_all_single(nccl_out, sv, outs, ins)
    n1.record(stream)
    torch.cuda.synchronize()
    nccl_ms = torch.tensor([n0.elapsed_time(n1) / args.steps], device="cuda")
    dist.all_reduce(nccl_ms, op=dist.ReduceOp.MAX)
    nccl_ms = float(nccl_ms.item())

    # e2e through the public API with host buffers (pinned H2D + D2H per step).
    # Pipelined like an application would: the send buffer is double-buffered
    # and step k+1's H2D runs on a copy stream while step k's exchange and its
    # D2H run on the compute stream (the receive region is reused, so a step's
    # D2H precedes the next exchange on that stream).  Every step's full H2D
    # and D2H lies inside the timed window; the first H2D starts after t0.
    host_send = torch.empty(send.numel(), dtype=torch.uint8, pin_memory=True)
    host_send.copy_(send)
    host_recv = torch.empty(int(D[:, rank].sum()), dtype=torch.uint8, pin_memory=True)
    dsend = [torch.empty_like(send), torch.empty_like(send)]
    cstream = torch.cuda.Stream()

    def e2e_run(K, e_start=None):
        h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        used = [None, None]  # event: the exchange that last read dsend[b] is done
        if e_start is not None:
            e_start.record(stream)
        cstream.wait_stream(stream)

        def h2d(k):
            b = k % 2
            if used[b] is not None:
                cstream.wait_event(used[b])
            with torch.cuda.stream(cstream):
                dsend[b].copy_(host_send, non_blocking=True)
                h2d_done[b].record(cstream)

        h2d(0)
        for k in range(K):
            b = k % 2
            if k + 1 < K:
                h2d(k + 1)
            stream.wait_event(h2d_done[b])
            r = comm.alltoallv(dsend[b], row)
            used[b] = torch.cuda.Event()
            used[b].record(stream)
            host_recv.copy_(r[: host_recv.numel()], non_blocking=True)

    for _ in range(2):
        e2e_run(2)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_run(args.steps, e0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    comm.check()
    # the last step's received bytes equal the device-path result
    if not torch.equal(host_recv[: nccl_out.numel()].cuda(), nccl_out):
        raise RuntimeError("e2e alltoallv result differs from NCCL all_to_all_single")

    ops = comm.plan.host_ops()
    fast_eg, fast_in = fast_wire_bytes(ops, G)
    direct_bn = int(max(D.sum(0).max(), D.sum(1).max()))
    t_roof = direct_bn / (PEER_GBS * 1e9)
    res = None
    if rank == 0:
        peaks, kind = measured_peaks()
        achieved = direct_bn / (exec_ms * 1e-3) / 1e9
        res = {
            "metric": "alltoallv algorithmic bandwidth (FAST schedule, P2P over NVSwitch; "
                      "whole job = algbw/GPU x N)",
            "value": round(total / (step_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8",
            "data": f"synthetic (Zipf {args.a2a_skew} traffic, seed {args.seed}, random payload)",
            "config": {"workload": "config2_alltoallv", "virtual_servers": f"{n}x{m}",
                       "total_bytes": total, "zipf_skew": args.a2a_skew},
            "bottleneck_gpu_bytes": direct_bn, "blocks_per_rank": args.blocks,
            "chunk_bytes": args.chunk,
            "l2": "payload per step %.0f MB; recv/staging are rewritten each step" % (total / 1e6),
            "algbw_gbps_per_gpu": round(algorithmic_bandwidth(total, G, step_ms * 1e-3) / 1e9, 3),
            "exec_kernel_ms": round(exec_ms, 4),
            "synth_and_plan_ms": round(step_ms - exec_ms, 4),
            "roofline": {"bound": "nvlink", "achieved": round(achieved, 2), "peak": PEER_GBS,
                         "unit": "GB/s", "frac": round(t_roof / (exec_ms * 1e-3), 4),
                         "traffic": None, "kernel": "exec_kernel",
                         "peak_source": "measured B200 peer copy per direction "
                                        "(B200_PROFILING.md); 900 GB/s nominal",
                         "frac_of_nominal": round(direct_bn / (NVLINK_NOMINAL * 1e9) / (exec_ms * 1e-3), 4),
                         "t_roof_us": round(t_roof * 1e6, 2),
                         "fast_one_tier_ceiling": round(direct_bn / max(fast_eg, fast_in), 4),
                         "fast_max_wire_bytes": max(fast_eg, fast_in),
                         "frac_step": round(t_roof / (step_ms * 1e-3), 4)},
            "nccl_all_to_all_single": {"ms": round(nccl_ms, 4),
                                       "value": round(total / (nccl_ms * 1e-3) / 1e9, 3),
                                       "unit": "GB/s", "nccl_env": nccl_env},
            "e2e": {"value": round(total / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": int(D[0].sum()) + 16,
                    "d2h_bytes_per_step": int(D[:, 0].sum()), "ms_per_step": round(e2e_ms, 4),
                    "path": "FastComm.alltoallv with pinned host send/recv (rank-0 bytes); "
                            "double-buffered send: step k+1's H2D on a copy stream overlaps "
                            "step k's exchange + D2H; max over ranks"},
            "gpu_launches": 6 * args.steps, "clocks": clk.summary(),
            "parity": "recv == NCCL all_to_all_single bytes on every rank",
            "peer_copy_peak_in_run": peaks_run,
        }
        if any(x is None for x in nvl_all):
            res["nvlink_counters"] = {
                "unavailable": "NVML NVLINK_THROUGHPUT_DATA_TX/RX fields return NOT_SUPPORTED, "
                               "GPM sampling fails and nvidia-smi nvlink -gt shows N/A on this "
                               "pool (tools/nvml_probe.py); see peer_copy_peak_in_run and the "
                               "per-rank globaltimer timeline (tools/exec_ranks.py)"}
        else:
            per = [{"rank": r, "tx_GB": round(x[0] / 1e9, 4), "rx_GB": round(x[1] / 1e9, 4),
                    "tx_GBps": round(x[0] / (x[2] * 1e-3) / 1e9, 1),
                    "rx_GBps": round(x[1] / (x[2] * 1e-3) / 1e9, 1)} for r, x in enumerate(nvl_all)]
            res["nvlink_counters"] = {
                "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX around the exec-only loop, per "
                          "exec call; GB/s over the rank's own exec-kernel event time",
                "per_rank": per,
                "max_rx_GBps_of_900": round(max(p["rx_GBps"] for p in per) / NVLINK_NOMINAL, 4),
                "wire_bytes_vs_plan": round(max(x[1] for x in nvl_all) / max(fast_in, 1), 4)}
        try:
            res["timeline"] = timeline_vs_model(D, n, m, tls, peaks_run)
        except Exception as exc:  # pragma: no cover - reported, not fatal
            res["timeline"] = {"error": repr(exc)[:200]}
        if peaks_run:
            pk = peaks_run["GBps"]["sm_copy"]
            res["roofline"]["frac_of_in_run_sm_peak"] = round(
                direct_bn / (pk * 1e9) / (exec_ms * 1e-3), 4)
            # what FAST can reach on ONE tier with SM stores: its own max wire
            # bytes per GPU at the measured SM-store peak
            t_fast = max(fast_eg, fast_in) / (pk * 1e9)
            res["roofline"]["fast_achievable_frac_of_nominal"] = round(
                direct_bn / (NVLINK_NOMINAL * 1e9) / t_fast, 4)
            res["roofline"]["exec_vs_fast_achievable"] = round(t_fast / (exec_ms * 1e-3), 4)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return res


NCCL_KNOBS = ("NCCL_NCHANNELS_PER_PEER", "NCCL_MIN_P2P_NCHANNELS", "NCCL_MAX_P2P_NCHANNELS",
              "NCCL_MIN_NCHANNELS", "NCCL_MAX_NCHANNELS", "NCCL_P2P_NVL_CHUNKSIZE",
              "NCCL_BUFFSIZE", "NCCL_NVLS_ENABLE", "NCCL_P2P_LEVEL")


def nccl_only(args, D: np.ndarray, rank: int, world: int) -> dict | None:
    """NCCL all_to_all_single alone on the config-2 traffic, with the NCCL
    environment of this process recorded (tools/nccl_sweep.sh varies it)."""
    ins, outs = D[rank].tolist(), D[:, rank].tolist()
    sv = torch.randint(0, 256, (int(D[rank].sum()),), dtype=torch.uint8, device="cuda")
    out = torch.empty(int(D[:, rank].sum()), dtype=torch.uint8, device="cuda")
    for _ in range(max(3, args.warmup)):
        dist.all_to_all_single(out, sv, outs, ins)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        dist.all_to_all_single(out, sv, outs, ins)
    b.record()
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    dist.destroy_process_group()
    if rank:
        return None
    return {"what": "nccl_all_to_all_single", "n_gpus": world, "ms": round(ms, 4),
            "GBps": round(int(D.sum()) / (ms * 1e-3) / 1e9, 2),
            "env": {k: os.environ[k] for k in NCCL_KNOBS if k in os.environ}}


def reference_alltoallv(args, world: int) -> dict:
    """Reference arm: tiersched.synthesize_fast (baseline/_ref) + the host
    memcpy alltoallv the schedule describes, on the host cores (rank 0)."""
    import sys

    from bench import REPO

    G = max(world, 2)
    n, m = topology_for(G, args.topo)
    D = demand(args, G)
    total = int(D.sum())
    ref = os.path.join(REPO, "baseline", "_ref")
    have = os.path.isdir(os.path.join(ref, "tiersched"))
    if have:
        sys.dont_write_bytecode = True
        sys.path.insert(0, ref)
        import tiersched as ts

        def synth():
            ts.synthesize_fast(ts.DemandMatrix(n, m, D.copy()), ts.Topology(n, m, 900e9, 900e9))
        kind = "reference"
    else:
        from oracle import oracle

        def synth():
            oracle.synthesize_batch(D, n, m)
        kind = "port"
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(0)
    sends = [rng.integers(0, 256, int(D[g].sum()), dtype=np.uint8) for g in range(G)]
    recvs = [np.empty(int(D[:, h].sum()), np.uint8) for h in range(G)]
    send_off = np.concatenate([np.zeros((G, 1), np.int64), np.cumsum(D, axis=1)[:, :-1]], axis=1)
    recv_off = np.concatenate([np.zeros((1, G), np.int64), np.cumsum(D, axis=0)[:-1, :]], axis=0)
    segs = [(g, h) for g in range(G) for h in range(G) if D[g, h] > 0]
    threads = os.cpu_count() or 1
    pool = ThreadPoolExecutor(threads)

    def copy_seg(gh):  # numpy releases the GIL while copying
        g, h = gh
        n_ = int(D[g, h])
        recvs[h][recv_off[g, h]:recv_off[g, h] + n_] = sends[g][send_off[g, h]:send_off[g, h] + n_]

    def step():
        t = time.perf_counter()
        synth()
        list(pool.map(copy_seg, segs))  # the alltoallv the schedule describes, every host thread
        return time.perf_counter() - t

    for _ in range(args.warmup):
        step()
    ts_ = [step() for _ in range(args.steps)]
    sec = sum(ts_) / len(ts_)
    val = total / sec / 1e9
    return {"impl": "reference",
            "metric": "alltoallv algorithmic bandwidth (FAST schedule, P2P over NVSwitch; "
                      "whole job = algbw/GPU x N)",
            "value": round(val, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": f"synthetic (Zipf {args.a2a_skew}, seed {args.seed})",
            "config": {"workload": "config2_alltoallv", "virtual_servers": f"{n}x{m}",
                       "total_bytes": total, "zipf_skew": args.a2a_skew},
            "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": threads,
                             "kind": kind,
                             "sample": "tiersched.synthesize_fast + host memcpy of every segment "
                                       f"(numpy, {threads} threads), full 256 MiB per step"},
            "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def run_moe(args) -> dict | None:
    """BASELINE config 3: Mixtral-style dispatch, E = 8 experts (--experts;
    E / N per GPU), top-2, 16k tokens x 4096 bf16 per GPU.  One step = gating -> histogram ->
    demand all-gather -> FAST synthesis -> pack -> P2P alltoallv -> unpack."""
    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.executor import FastComm
    from paper_2505_09764_b200.moe import MoEDispatch

    nccl_env = _tune_nccl()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, m = topology_for(world, args.topo)
    T, hidden = args.tokens, args.hidden
    RB = hidden * 2
    cap = T * 2 * RB * 3  # generous: the hot experts' rank can receive 3x its share
    comm = FastComm(Topology(n, m), recv_bytes=cap, staging_bytes=cap, blocks=args.blocks,
                    chunk_bytes=args.chunk)
    E = args.experts if args.experts % world == 0 else world
    disp = MoEDispatch(comm, T, RB, num_experts=E)
    gen = torch.Generator(device="cuda").manual_seed(7 + rank)
    tokens = torch.randn(T, hidden, dtype=torch.bfloat16, device="cuda", generator=gen)
    stream = torch.cuda.current_stream()
    recv = disp.dispatch(tokens, seed=args.seed)
    torch.cuda.synchronize()
    comm.check()
    Dg = comm.demand().cpu().numpy() + np.diag(comm.self_sizes().cpu().numpy())
    # NCCL bar: all_to_all_single of the same packed buffer (self included)
    ins, outs = Dg[rank].tolist(), Dg[:, rank].tolist()
    nsend = disp.send[: int(Dg[rank].sum())]
    nccl_out = torch.empty(int(Dg[:, rank].sum()), dtype=torch.uint8, device="cuda")
    dist.all_to_all_single(nccl_out, nsend, outs, ins)
    torch.cuda.synchronize()
    ok = torch.equal(recv[: nccl_out.numel()], nccl_out)
    okt = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(okt)
    if int(okt.item()) != 0:
        raise RuntimeError("MoE expert input differs from NCCL all_to_all_single")
    for _ in range(args.warmup):
        disp.dispatch(tokens, seed=args.seed)
    torch.cuda.synchronize()
    dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            disp.dispatch(tokens, seed=args.seed)
        t1.record(stream)
        torch.cuda.synchronize()
    comm.check()
    ms = torch.tensor([t0.elapsed_time(t1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # fused pack -> send (row-mapped executor source): same expert input, no
    # packed send buffer written or read
    fdisp = MoEDispatch(comm, T, RB, fused_pack=True, num_experts=E)
    frecv = fdisp.dispatch(tokens, seed=args.seed)
    torch.cuda.synchronize()
    comm.check()
    okf = torch.tensor([0 if torch.equal(frecv[: nccl_out.numel()], nccl_out) else 1],
                       device="cuda")
    dist.all_reduce(okf)
    if int(okf.item()) != 0:
        raise RuntimeError("fused-pack MoE expert input differs from NCCL all_to_all_single")
    for _ in range(args.warmup):
        fdisp.dispatch(tokens, seed=args.seed)
    torch.cuda.synchronize()
    dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        fdisp.dispatch(tokens, seed=args.seed)
    f1.record(stream)
    torch.cuda.synchronize()
    comm.check()
    fms = torch.tensor([f0.elapsed_time(f1) / args.steps], device="cuda")
    dist.all_reduce(fms, op=dist.ReduceOp.MAX)
    fms = float(fms.item())
    disp.dispatch(tokens, seed=args.seed)  # the combine below uses disp's forward state
    torch.cuda.synchronize()
    # NCCL path: our route + pack, NCCL alltoall (no FAST), timed the same way
    for _ in range(args.warmup):
        disp.route(args.seed)
        disp.pack(tokens)
        dist.all_to_all_single(nccl_out, nsend, outs, ins)
    torch.cuda.synchronize()
    dist.barrier()
    n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0.record(stream)
    for _ in range(args.steps):
        disp.route(args.seed)
        disp.pack(tokens)
        dist.all_to_all_single(nccl_out, nsend, outs, ins)
    n1.record(stream)
    torch.cuda.synchronize()
    nms = torch.tensor([n0.elapsed_time(n1) / args.steps], device="cuda")
    dist.all_reduce(nms, op=dist.ReduceOp.MAX)
    nms = float(nms.item())
    # combine (the second alltoallv of the layer): identity experts
    expert_out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    expert_out.copy_(recv[:cap])
    wts = torch.rand(T, 2, dtype=torch.float32, device="cuda")
    comb_out = torch.empty(T, hidden, dtype=torch.bfloat16, device="cuda")
    for _ in range(args.warmup):
        disp.combine(expert_out, wts, comb_out)
    torch.cuda.synchronize()
    dist.barrier()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(args.steps):
        disp.combine(expert_out, wts, comb_out)
    c1.record(stream)
    torch.cuda.synchronize()
    comm.check()
    cms = torch.tensor([c0.elapsed_time(c1) / args.steps], device="cuda")
    dist.all_reduce(cms, op=dist.ReduceOp.MAX)
    cms = float(cms.item())
    D = comm.demand().cpu().numpy()
    cross = int(D.sum())
    bn = int(max(D.sum(0).max(), D.sum(1).max()))
    res = None
    if rank == 0:
        res = {"metric": "MoE dispatch throughput (gating -> histogram -> schedule -> pack -> "
                         "alltoallv -> unpack; whole job)",
               "value": round(T * world / (fms * 1e-3), 1), "unit": "tokens/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(fms, 4), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "bf16 payload (bytes moved as u8)",
               "data": "synthetic tokens, deterministic integer top-2 gating",
               "config": {"workload": "config3_moe_dispatch", "virtual_servers": f"{n}x{m}",
                          "experts": E, "experts_per_gpu": E // world, "top_k": 2,
                          "tokens_per_gpu": T,
                          "hidden": hidden, "cross_gpu_bytes": cross,
                          "bottleneck_gpu_bytes": bn},
               "t_roof_us": round(bn / (PEER_GBS * 1e9) * 1e6, 1),
               "frac_of_alltoallv_roofline": round(bn / (PEER_GBS * 1e9) / (fms * 1e-3), 4),
               "pack": "fused into the executor's source reads (row map, no send buffer)",
               "packed_path": {"ms": round(ms, 4),
                               "value": round(T * world / (ms * 1e-3), 1), "unit": "tokens/s",
                               "what": "same dispatch with the pack kernel materialising "
                                       "the send buffer",
                               "parity": "expert input == NCCL all_to_all_single"},
               "combine_ms": round(cms, 4),
               "layer_dispatch_plus_combine_ms": round(fms + cms, 4),
               "nccl_path": {"ms": round(nms, 4),
                             "value": round(T * world / (nms * 1e-3), 1), "unit": "tokens/s",
                             "what": "same route+pack kernels + NCCL all_to_all_single",
                             "nccl_env": nccl_env},
               "clocks": clk.summary(),
               "parity": "expert input == NCCL all_to_all_single of the packed buffer"}
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return res


def run_sweep(args) -> dict | None:
    """BASELINE config 4: per-step shifting hotspot (GPU k mod N is hot, its row
    and column x8 over a uniform base), per-GPU send size swept 1 KiB -> 1 GiB
    in x4 steps.  Every step has a new traffic matrix, so the demand
    all-gather + synthesis + plan are on the critical path; reports the
    end-to-end step time, the exec-kernel time and NCCL all_to_all_single."""
    from paper_2505_09764_b200 import Topology, workloads
    from paper_2505_09764_b200.executor import FastComm

    _tune_nccl()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, m = topology_for(world, args.topo or ("4x2" if world == 8 else None))
    t = Topology(n, m)
    sizes = [1024 * 4 ** k for k in range(11) if 1024 * 4 ** k <= args.sweep_max]
    steps = max(args.steps, world)  # every GPU is hot at least once
    mats = {}
    cap = stg = 0
    for S in sizes:
        ds = []
        for it in range(steps):
            mean = max(1, S // (world - 1) // 2)  # uniform base: mean row ~ S
            d = workloads.gen_hotspot(1000 * it + 7, t, mean, hot=it % world, factor=8).sizes
            ds.append(d)
            cap = max(cap, int(d.sum(0).max()), int(d.sum(1).max()))
        mats[S] = ds
    cap += 4096
    comm = FastComm(t, recv_bytes=cap, staging_bytes=2 * cap + (4 << 20), blocks=args.blocks,
                    chunk_bytes=args.chunk)
    send = torch.randint(0, 256, (cap,), dtype=torch.uint8, device="cuda")
    nccl_out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    rows_dev = {S: [torch.from_numpy(d[rank].copy()).cuda() for d in mats[S]] for S in sizes}
    table = []
    for S in sizes:
        ds, rows = mats[S], rows_dev[S]
        for it in range(min(args.warmup, steps)):
            comm.alltoallv(send, rows[it])
        torch.cuda.synchronize()
        dist.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for it in range(steps):
            comm.alltoallv(send, rows[it], exec_events=ev[it])
        t1.record(stream)
        torch.cuda.synchronize()
        comm.check()
        fast_ms = t0.elapsed_time(t1) / steps
        exec_ms = sum(a.elapsed_time(b) for a, b in ev) / steps
        for it in range(min(args.warmup, steps)):
            d = ds[it]
            dist.all_to_all_single(nccl_out[: int(d[:, rank].sum())], send[: int(d[rank].sum())],
                                   d[:, rank].tolist(), d[rank].tolist())
        torch.cuda.synchronize()
        dist.barrier()
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0.record(stream)
        for it in range(steps):
            d = ds[it]
            dist.all_to_all_single(nccl_out[: int(d[:, rank].sum())], send[: int(d[rank].sum())],
                                   d[:, rank].tolist(), d[rank].tolist())
        n1.record(stream)
        torch.cuda.synchronize()
        nccl_ms = n0.elapsed_time(n1) / steps
        v = torch.tensor([fast_ms, exec_ms, nccl_ms], device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        fast_ms, exec_ms, nccl_ms = (float(x) for x in v.tolist())
        tot = sum(int(d.sum()) for d in ds) / steps
        bn = sum(int(max(d.sum(0).max(), d.sum(1).max())) for d in ds) / steps
        table.append({"bytes_per_gpu": S, "fast_us": round(fast_ms * 1e3, 2),
                      "exec_us": round(exec_ms * 1e3, 2), "nccl_us": round(nccl_ms * 1e3, 2),
                      "fast_GBps": round(tot / (fast_ms * 1e-3) / 1e9, 3),
                      "nccl_GBps": round(tot / (nccl_ms * 1e-3) / 1e9, 3),
                      "frac_roofline_exec": round(bn / (PEER_GBS * 1e9) / (exec_ms * 1e-3), 4)})
    res = None
    if rank == 0:
        last = table[-1]
        res = {"metric": "alltoallv algbw under a shifting hotspot (config 4; whole job, "
                         "synthesis on the critical path every step)",
               "value": last["fast_GBps"], "unit": "GB/s", "n_gpus": world, "steps": steps,
               "warmup": args.warmup, "ms_per_step": round(last["fast_us"] / 1e3, 4),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
               "data": "synthetic hotspot traffic (x8 row/col of GPU k mod N at step k)",
               "config": {"workload": "config4_hotspot_sweep", "virtual_servers": f"{n}x{m}",
                          "sizes": [r["bytes_per_gpu"] for r in table]},
               "sweep": table}
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    return res
