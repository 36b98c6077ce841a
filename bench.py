#!/usr/bin/env python
"""Benchmark of the FAST All-to-All(v) hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 (default): BASELINE config 5, schedule-synthesis scaling -- one step is
synthesize_fast over a batch of 1000 Zipf(0.8) traffic matrices of
n = 128 virtual servers x 8 GPUs (the largest single-GPU configuration),
inputs resident in HBM.  N > 1 (torchrun, one rank per GPU): the alltoallv
workload (BASELINE config 2 shape) executed by the P2P stage executor over
NVSwitch (see bench_alltoallv in this file).

Rank 0 prints ONE JSON line.  ``--impl reference`` times the reference's own
CPU implementation (tiersched from baseline/_ref, else the C oracle port) on
the same config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

# the e2e path streams batches over 2 x 8 chunk streams: give each its own
# hardware queue (must be set before the CUDA context exists)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# rank 0 prints exactly one JSON line: keep NCCL's version banner off stdout
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

HBM_FALLBACK_GBS = 6650.0


def measured_peaks() -> tuple[dict, str]:
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": HBM_FALLBACK_GBS}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        rows = []
        if self.path and os.path.exists(self.path):
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].isdigit():
                    rows.append(parts)
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": int(statistics.median(busy)), "sm_max_mhz": int(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# config 5: batched schedule synthesis on 1 GPU

def synth_inputs(args, device):
    from paper_2505_09764_b200 import workloads

    G = args.n * args.m
    return workloads.zipf_batch_device(range(args.batch), G, args.skew, args.total, device)


def algorithmic_bytes_decompose(n: int, n_raw) -> int:
    # read server matrix, write aux, write each raw stage (weight + perm + bytes)
    return int(sum(16 * n * n + int(k) * (8 + 9 * n) for k in n_raw))


# Dependent-chain floor of one DFS step of the decomposition (cycles):
# ld.shared.v4 (34.6) -> and -> bfind (~16) -> mad -> 2 x selp -> next load,
# measured with tools/op_lat.cu / tools/chase2_micro.cu (profiles/README.md).
DFS_STEP_FLOOR_CYCLES = 70.0

SUBSET_KEYS = ("balanced", "server", "move_count", "moves", "common_sum", "aux", "n_raw",
               "stage_weight", "stage_perm", "stage_bytes", "n_stages", "stage_order", "status")


def device_subset(bufs, k: int) -> dict:
    """Host copy of the first k matrices of a SynthBuffers (parity check)."""
    return {key: getattr(bufs, key)[:k].cpu().numpy() for key in SUBSET_KEYS}


def compare_with_oracle(ref: dict, b: int, got: dict, what: str) -> None:
    """Bit-exact comparison of one matrix's schedule with the oracle's."""
    from paper_2505_09764_b200.schedule import MOVE_DTYPE

    k, s = int(ref["n_raw"][b]), int(ref["n_stages"][b])
    checks = [("status", got["status"] == ref["status"][b]),
              ("balanced", np.array_equal(got["balanced"], ref["balanced"][b])),
              ("server", np.array_equal(got["server"], ref["server"][b])),
              ("move_count", np.array_equal(got["move_count"], ref["move_count"][b])),
              ("common_sum", got["common_sum"] == ref["common_sum"][b]),
              ("aux", np.array_equal(got["aux"], ref["aux"][b])),
              ("n_raw", got["n_raw"] == k), ("n_stages", got["n_stages"] == s),
              ("stage_weight", np.array_equal(got["stage_weight"][:k], ref["stage_weight"][b, :k])),
              ("stage_perm", np.array_equal(got["stage_perm"][:k], ref["stage_perm"][b, :k])),
              ("stage_bytes", np.array_equal(got["stage_bytes"][:k], ref["stage_bytes"][b, :k])),
              ("stage_order", np.array_equal(got["stage_order"][:s], ref["stage_order"][b, :s]))]
    mv = got["moves"].view(MOVE_DTYPE).reshape(ref["moves"].shape[1:])
    cnt = ref["move_count"][b]
    used = np.arange(mv.shape[1])[None, :] < cnt[:, None]
    checks.append(("moves", np.array_equal(mv[used], ref["moves"][b][used])))
    bad = [name for name, ok in checks if not bool(ok)]
    if bad:
        raise RuntimeError(f"PARITY FAILURE ({what}, matrix {b}): {bad}")


def bench_synth(args) -> dict:
    import torch

    from paper_2505_09764_b200 import _lib, synth

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = _lib.load()
    n, m, B = args.n, args.m, args.batch
    G, T = n * m, n * (n - 1)
    D = synth_inputs(args, dev)
    # device-resident product layout (balanced matrix, moves, raw stages with
    # per-edge bytes, sort order): what the executor and other device
    # consumers read.  The e2e leg below adds the host transport format (aux
    # run-out table + compact balanced tiles) and times it separately.
    # `inflight` batches are processed concurrently (rotating buffer sets on
    # their own streams): one batch of 1000 chains leaves the SM schedulers
    # ~60 % idle (7 latency-bound warps per SM); decomposition throughput
    # saturates at ~14.6 K matrices/s with >= 2000 chains resident
    # (profiles/r2_inflight.log), and 3 in flight also hide each batch's
    # balance and sort behind the others' decompositions
    depth = max(1, args.inflight)
    sets = [synth.SynthBuffers(B, n, m, dev) for _ in range(depth)]
    streams = [torch.cuda.Stream(dev) for _ in range(depth)]
    stream = torch.cuda.current_stream()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def make_events(k):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(k)]
        for row in evs:
            for e in row:
                e.record(stream)  # materialise the handles
        return evs

    def step(k, ev_row=None):
        arr = None
        if ev_row is not None:
            arr = (ctypes.c_void_p * 4)(*[e.cuda_event for e in ev_row[:4]])
        st = streams[k % depth]
        rc = lib.fast_synth_batch_ev(P(D), B, n, m, ctypes.byref(sets[k % depth].struct),
                                     ctypes.c_void_p(st.cuda_stream), arr)
        _lib.check_rc(rc, "fast_synth_batch_ev")

    def run_steps(K, evs=None):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for st in streams:
            st.wait_event(t0)
        for k in range(K):
            step(k, evs[k] if evs is not None else None)
        for st in streams:
            stream.wait_stream(st)
        t1.record(stream)
        return t0, t1

    run_steps(max(args.warmup, depth))
    torch.cuda.synchronize()
    for bufs in sets:
        status = bufs.status.cpu()
        if int(status.abs().max()) != 0:
            raise RuntimeError(f"synthesis failed on {int((status != 0).sum())} matrices")

    evs = make_events(args.steps)
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        t0, t1 = run_steps(args.steps, evs)
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    names = ("balance_kernel", "decompose_kernel", "sort_kernel")
    per = {k: 0.0 for k in names}
    for row in evs:
        for i, k in enumerate(names):
            per[k] += row[i].elapsed_time(row[i + 1])
    per = {k: v / args.steps for k, v in per.items()}
    ms_step = total_ms / args.steps
    # one batch alone (nothing else in flight): the batch latency
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat_ev = make_events(1)[0]
    a0.record(stream)
    rc = lib.fast_synth_batch_ev(P(D), B, n, m, ctypes.byref(sets[0].struct),
                                 ctypes.c_void_p(stream.cuda_stream),
                                 (ctypes.c_void_p * 4)(*[e.cuda_event for e in lat_ev]))
    _lib.check_rc(rc, "fast_synth_batch_ev")
    a1.record(stream)
    torch.cuda.synchronize()
    batch_alone_ms = a0.elapsed_time(a1)
    alone = {k: lat_ev[i].elapsed_time(lat_ev[i + 1]) for i, k in enumerate(names)}
    bufs = sets[0]
    n_raw = bufs.n_raw.cpu().tolist()
    P_CHECK = min(64, B)
    dev_sub = device_subset(bufs, P_CHECK)
    d2h_device_layout = int(bufs.output_nbytes())

    peaks, peak_kind = measured_peaks()
    hbm = float(peaks["hbm_gbs"])
    alg = {"balance_kernel": 16 * G * G * B,
           "decompose_kernel": algorithmic_bytes_decompose(n, n_raw),
           "sort_kernel": int(sum(8 * 2 * k for k in n_raw))}
    traffic = None
    tf = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(f"decompose_kernel/n{n}_m{m}_B{B}")
    sm_hz = None
    try:
        sm_hz = torch.cuda.get_device_properties(0).clock_rate * 1e3
    except Exception:
        pass
    if not sm_hz:
        sm_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peels = sum(n_raw) / len(n_raw)
    # The dominant kernel (decompose, 92 % of a batch) is a dependent
    # shared-memory chain, not an HBM stream: its roofline is cycles per DFS
    # step against the chain floor, filled in below from
    # the oracle's DFS step count of the checked matrices.  Per-kernel device
    # times come from the batch run alone (the in-flight overlap stretches
    # every kernel's own event window).
    bal_gbs = alg["balance_kernel"] / (alone["balance_kernel"] * 1e-3) / 1e9
    dec_gbs = alg["decompose_kernel"] / (alone["decompose_kernel"] * 1e-3) / 1e9
    roofline = {"bound": "latency", "kernel": "decompose_kernel",
                "achieved": None, "peak": DFS_STEP_FLOOR_CYCLES,
                "unit": "cycles per DFS step (whole kernel; lower is better, frac = peak/achieved)",
                "frac": None, "traffic": traffic,
                "algorithmic_bytes": alg["decompose_kernel"],
                "kernel_ms_batch_alone": {k: round(v, 4) for k, v in alone.items()},
                "kernel_ms_in_flight": {k: round(v, 4) for k, v in per.items()},
                "decompose_cycles_per_peel": round(alone["decompose_kernel"] * 1e-3 * sm_hz / peels,
                                                   1),
                "hbm_view": {"bound": "hbm", "peak": hbm, "unit": "GB/s",
                             "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                             "decompose_kernel_gbs": round(dec_gbs, 1),
                             "decompose_kernel_frac": round(dec_gbs / hbm, 5),
                             "balance_kernel_gbs": round(bal_gbs, 1),
                             "balance_kernel_frac": round(bal_gbs / hbm, 4),
                             "note": "balance is the HBM-bound kernel; decompose's HBM fraction is "
                                     "reported for completeness only"}}

    # ---- e2e: host (pinned) D -> device -> synth -> compact result -> host,
    # through the public host-buffer API (HostSynthPipeline: chunked, copies
    # overlapped with kernels).  Headline: a stream of batches (batch k+1's
    # H2D and kernels enqueued before batch k completes; every batch's full
    # H2D and D2H inside the timed region).  Also reported: one synchronous
    # call (latency of a single batch).
    e2e = None
    hs = Dh = None
    if not args.no_e2e:
        Dh = torch.empty(D.shape, dtype=D.dtype, pin_memory=True)
        Dh.copy_(D)
        del bufs, sets
        torch.cuda.empty_cache()
        depth = max(1, args.e2e_depth)
        pipe = synth.HostSynthPipeline(B, n, m, chunk=args.e2e_chunk, depth=depth)
        nout = max(2, depth)
        outs = [synth.HostSchedules(B, n, m) for _ in range(nout)]
        pipe.run([Dh] * nout, outs)  # sizes the host value buffers
        K = max(4, args.steps)
        Wb = max(args.warmup, nout)
        # one continuous stream of Wb + K batches (at most `depth` in flight);
        # the timed window runs from the completion of the last warm-up batch
        # to the completion of the K-th timed batch, so it holds K batches'
        # worth of H2D, kernels and D2H in steady state (the pipeline's fill
        # is the warm-up's, reported apart as fill_ms)
        torch.cuda.synchronize()
        pending, comp = [], []
        t_sub0 = time.perf_counter()

        def complete():
            h = pipe.result(pending.pop(0))
            comp.append(time.perf_counter())
            if int(h.status.abs().max()) != 0:
                raise RuntimeError("e2e synthesis reported failures")
            return h

        for t in range(Wb + K):
            pending.append(pipe.submit(Dh, outs[t % nout]))
            if len(pending) >= depth:
                hs = complete()
        while pending:
            hs = complete()
        ems = (comp[Wb + K - 1] - comp[Wb - 1]) * 1e3 / K
        fill_ms = (comp[0] - t_sub0) * 1e3
        torch.cuda.synchronize()
        t1h = time.perf_counter()
        pipe.result(pipe.submit(Dh, outs[0]))
        sync_ms = (time.perf_counter() - t1h) * 1e3
        hs = outs[0]
        del pipe
        e2e = {"value": round(B / (ems * 1e-3), 3), "unit": "matrices/s",
               "h2d_bytes_per_step": int(Dh.numel() * 8), "d2h_bytes_per_step": int(hs.nbytes()),
               "ms_per_step": round(ems, 3), "steps": K, "warmup_batches": Wb,
               "batches_in_flight": depth, "fill_ms": round(fill_ms, 3),
               "sync_ms_per_batch": round(sync_ms, 3),
               "sync_value": round(B / (sync_ms * 1e-3), 3),
               "d2h_full_device_layout_bytes": d2h_device_layout,
               "path": f"HostSynthPipeline (public host-buffer API: C-ABI fast_synth_batch + "
                       f"fast_compact_batch per {args.e2e_chunk}-matrix chunk), pinned host D in, "
                       "compact schedule out (HostSchedules: moves, stages, aux run-out table, "
                       "changed cells of the balanced tiles); one continuous stream of "
                       "warm-up + K batches, timed (wall clock, host sync on each result) from "
                       "the last warm-up batch's completion to the K-th timed batch's: K "
                       "batches' H2D + D2H in steady state; fill_ms: first batch's latency in "
                       "the stream; sync_*: one synchronous call"}

    cpu, parity = None, None
    if not args.no_cpu_baseline:
        cpu, ref = cpu_baseline_synth(args, D)
        k_chk = min(P_CHECK, int(ref["n_raw"].shape[0]))
        for b in range(k_chk):
            got = {key: dev_sub[key][b] for key in SUBSET_KEYS}
            compare_with_oracle(ref, b, got, "device path")
            if hs is not None:
                p = hs.packed(b, Dh[b].numpy())
                compare_with_oracle(ref, b, dict(
                    status=p.status, balanced=p.balanced, server=p.server,
                    move_count=p.move_count, moves=p.moves.view(np.int64).reshape(-1, 2),
                    common_sum=p.common_sum, aux=p.aux, n_raw=p.n_raw, n_stages=p.n_stages,
                    stage_weight=p.stage_weight, stage_perm=p.stage_perm,
                    stage_bytes=p.stage_bytes, stage_order=p.stage_order), "e2e compact path")
        steps_mean = cpu.pop("_dfs_steps_mean")
        parity = {"parity_checked": k_chk, "against": "oracle/fast_oracle.c (pinned to tiersched "
                  "by tests/golden/headline_digests.json)", "paths": ["device", "e2e"] if hs is not None
                  else ["device"], "result": "bit-exact"}
        cyc = alone["decompose_kernel"] * 1e-3 * sm_hz / steps_mean
        roofline["achieved"] = round(cyc, 1)
        roofline["frac"] = round(DFS_STEP_FLOOR_CYCLES / cyc, 4)
        roofline["chain"] = {
            "bound": "dependent shared-memory chain (Kuhn DFS)", "kernel": "decompose_kernel",
            "dfs_steps_per_matrix": round(steps_mean, 1),
            "steps_source": f"oracle DFS step counter on the {k_chk} checked matrices",
            "cycles_per_step": round(cyc, 1), "floor_cycles_per_step": DFS_STEP_FLOOR_CYCLES,
            "frac": round(DFS_STEP_FLOOR_CYCLES / cyc, 4),
            "note": "whole-kernel cycles of one batch alone (1000 chains resident, kernel time = "
                    "slowest chain) per DFS step; the floor is one step's dependent "
                    "LDS->and->bfind->mad->selp chain"}

    out = {
        "metric": "schedule synthesis throughput (FAST synthesize_fast, batch of 1000 traffic "
                  "matrices, config 5)",
        "value": round(B / (ms_step * 1e-3), 3), "unit": "matrices/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "us_per_matrix": round(ms_step * 1e3 / B, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (Zipf 0.8 traffic matrices, seeds 0..B-1, generated on device)",
        "config": {"workload": "config5_synthesis", "n_servers": n, "gpus_per_server": m,
                   "batch": B, "zipf_skew": args.skew, "total_bytes": args.total},
        "l2": "inputs larger than L2 (D batch = %.1f GB)" % (B * G * G * 8 / 1e9)
              if B * G * G * 8 > 126e6 else "inputs within L2",
        "inflight_batches": depth,
        "batch_alone_ms": round(batch_alone_ms, 3),
        "batch_alone_kernel_ms": {k: round(v, 4) for k, v in alone.items()},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": 3 * args.steps, "clocks": clk.summary(),
        "stages_per_matrix_mean": round(peels, 1),
    }
    if parity is not None:
        out["parity"] = parity
        out["parity_checked"] = parity["parity_checked"]
    if not args.no_latency:
        out["latency"] = single_matrix_latency(args)
    return out


def single_matrix_latency(args) -> dict:
    """Per-matrix synthesis LATENCY at 1 GPU (one matrix per call, B = 1),
    n = 16..128 x 8, Zipf 0.8: device time of fast_synth_batch from CUDA
    events, median of a few calls."""
    import torch

    from paper_2505_09764_b200 import _lib, synth, workloads

    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sh = ctypes.c_void_p(stream.cuda_stream)
    res = {}
    # the paper's own synthesis times (C++ on a Xeon 8468):
    # 4x8 25 us, 8x8 221 us, 12x8 805 us, 40x8 77 ms
    paper = {4: 25.0, 8: 221.0, 12: 805.0, 40: 77000.0}
    for n in (4, 8, 12, 16, 32, 40, 64, 128):
        G = n * args.m
        D = workloads.zipf_batch_device([0], G, args.skew, args.total, torch.device("cuda", 0))
        bufs = synth.SynthBuffers(1, n, args.m, D.device)

        def call(st):
            _lib.check_rc(lib.fast_synth_batch(ctypes.c_void_p(D.data_ptr()), 1, n, args.m,
                                               ctypes.byref(bufs.struct),
                                               ctypes.c_void_p(st.cuda_stream)),
                          "fast_synth_batch")

        # calls replayed from a CUDA graph (as the executor issues them), so
        # host launch gaps do not count as device latency
        reps = 20 if n <= 64 else 2
        call(stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                call(torch.cuda.current_stream())
        times = []
        for r in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b) / reps)
        res[f"n{n}"] = {"us": round(min(times) * 1e3, 1), "stages": int(bufs.n_raw.item())}
        del g
        if n in paper:
            res[f"n{n}"]["paper_cpu_us"] = paper[n]
    return {"what": "one matrix per call (B=1), device time per call of a CUDA graph of "
                    "back-to-back calls, best of 3; paper_cpu_us: the paper's "
                    "published synthesis time for that server count (PAPER.md:550-551)",
            "unit": "us", **res}


def cpu_baseline_synth(args, D, budget_s: float = 12.0) -> tuple[dict, dict]:
    """C oracle port (single thread) on a bounded sample of the same batch.
    Returns the baseline line and the oracle's results (the parity check of
    the timed batch)."""
    from oracle import oracle

    n, m = args.n, args.m
    Dh = D[: min(64, D.shape[0])].cpu().numpy()
    oracle.synthesize_batch(Dh[:1], n, m)  # load / warm
    oracle.dfs_counters(reset=True)
    done, t0, outs = 0, time.perf_counter(), []
    while done < Dh.shape[0]:
        outs.append(oracle.synthesize_batch(Dh[done:done + 1], n, m))
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    steps, _ = oracle.dfs_counters(reset=True)
    ref = {k: np.concatenate([o[k] for o in outs]) for k in outs[0]}
    return ({"value": round(done / el, 4), "unit": "matrices/s", "cores": 1, "kind": "port",
             "sample": f"{done} matrices of the benchmark batch (n={n}, m={m}), "
                       f"C restatement oracle/fast_oracle.c, 1 thread, {el:.1f} s",
             "_dfs_steps_mean": steps / done}, ref)


# ---------------------------------------------------------------------------
# reference arm: tiersched (baseline/_ref) on the host cores

def _ref_worker_init(path):
    sys.dont_write_bytecode = True
    sys.path.insert(0, path)


def _ref_synth_one(task):
    import numpy as np
    import tiersched as ts

    n, m, sizes = task
    d = ts.DemandMatrix(n_servers=n, gpus_per_server=m, sizes=np.asarray(sizes, np.int64))
    t = ts.Topology(n, m, 900e9, 900e9)
    t0 = time.perf_counter()
    ts.synthesize_fast(d, t)
    return time.perf_counter() - t0


def reference_synth(args) -> dict:
    import multiprocessing as mp

    from paper_2505_09764_b200 import workloads

    ref = os.path.join(REPO, "baseline", "_ref")
    have_ref = os.path.isdir(os.path.join(ref, "tiersched"))
    cores = os.cpu_count() or 1
    n, m = args.n, args.m
    G = n * m
    sample = [workloads.zipf_sizes(s, G, args.skew, args.total) for s in range(cores)]
    if have_ref:
        pool = mp.get_context("spawn").Pool(cores, initializer=_ref_worker_init, initargs=(ref,))

        def run_step():
            t0 = time.perf_counter()
            pool.map(_ref_synth_one, [(n, m, s) for s in sample])
            return time.perf_counter() - t0
        kind, what = "reference", "tiersched.synthesize_fast (baseline/_ref, unmodified Python)"
    else:
        from oracle import oracle
        import numpy as np

        arr = np.stack(sample)

        def run_step():
            t0 = time.perf_counter()
            oracle.synthesize_batch(arr, n, m)
            return time.perf_counter() - t0
        kind, what, cores = "port", "oracle/fast_oracle.c (1 thread)", 1
    for _ in range(args.warmup):
        run_step()
    times = [run_step() for _ in range(args.steps)]
    tot = sum(times)
    value = len(sample) * args.steps / tot
    if have_ref:
        pool.close()
    return {
        "impl": "reference",
        "metric": "schedule synthesis throughput (FAST synthesize_fast, batch of 1000 traffic "
                  "matrices, config 5)",
        "value": round(value, 5), "unit": "matrices/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (Zipf 0.8 traffic matrices)",
        "config": {"workload": "config5_synthesis", "n_servers": n, "gpus_per_server": m,
                   "batch": args.batch, "zipf_skew": args.skew, "total_bytes": args.total},
        "cpu_baseline": {"value": round(value, 5), "unit": "matrices/s", "cores": cores,
                         "kind": kind,
                         "sample": f"{len(sample)} matrices per step, one per worker process; {what}"},
        "e2e": {"value": round(value, 5), "unit": "matrices/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


# ---------------------------------------------------------------------------

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("auto", "synth", "alltoallv", "moe", "sweep"),
                    default="auto")
    ap.add_argument("--sweep-max", type=int, default=1 << 30)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1000)
    ap.add_argument("--skew", type=float, default=0.8)
    ap.add_argument("--total", type=int, default=2**34)
    ap.add_argument("--topo", default=None, help="alltoallv virtual servers, e.g. 4x2")
    ap.add_argument("--a2a-skew", type=float, default=1.2)
    ap.add_argument("--a2a-total", type=int, default=268_435_456)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--blocks", type=int, default=128)
    ap.add_argument("--chunk", type=int, default=1024 * 1024)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--nccl-only", action="store_true")
    ap.add_argument("--inflight", type=int, default=3,
                    help="config 5: batches in flight (rotating buffer sets / streams)")
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--e2e-chunk", type=int, default=125)
    ap.add_argument("--e2e-depth", type=int, default=2, help="HostSynthPipeline buffer sets")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    workload = args.workload
    if workload == "auto":
        workload = "synth" if args.gpus == 1 and world == 1 else "alltoallv"

    if workload == "synth":
        if rank != 0:
            return
        res = reference_synth(args) if args.impl == "reference" else bench_synth(args)
        print(json.dumps(res), flush=True)
        return
    from bench_exec import run as run_exec
    from bench_exec import run_moe, run_sweep

    if workload == "moe":
        res = run_moe(args)
    elif workload == "sweep":
        res = run_sweep(args)
    else:
        res = run_exec(args, workload)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
