"""Analytical cost model on the GPU.

Drop-in for the reference's model module and its neighbours:
  simulate_fast, simulate_spreadout, step_cost, intra_phase_time, Timeline
      /root/reference/pkg/src/tiersched/simulate.py:38-242
  spreadout_stages, spreadout_completion_units, spreadout_intra
      spreadout.py:19-67;  synthesize_spreadout, SpreadoutSchedule  pipeline.py:43-69
  optimal_time, fast_worstcase_time, ratio_bound, intra_assumption_holds,
  bounds_report, BoundsReport                                    bounds.py:17-120
  split_deliveries, stage_redistribution                         balance.py:177-265

The per-schedule model (every simulate_* call and the bounds) runs in the
batched sm_100a kernel csrc/sim.cu through fast_simulate_batch, in the
reference's IEEE double operation order, so results are bit-identical
(tests/test_simulate.py against the reference's own outputs).
simulate_batch() evaluates a whole SynthBuffers batch straight from the
device-resident synthesis output.  step_cost / intra_phase_time /
split_deliveries / stage_redistribution / spreadout_intra are scalar or
list-building helpers on host objects and stay host-side.
"""

from __future__ import annotations

import ctypes
import warnings
from collections.abc import Iterable, Mapping, Sequence
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._abi_ext import FastSimIn, FastSimOut, FastSimTopo
from .model import (
    DemandMatrix,
    InternalInvariantError,
    ServerMatrix,
    Topology,
    ValidationError,
    max_rc,
    reduce_to_server_level,
)
from .schedule import BalancePlan, IntraMove, PermutationStage

__all__ = [
    "BoundsReport", "SimBuffers", "SpreadoutSchedule", "Timeline", "bounds_report",
    "fast_worstcase_time", "intra_assumption_holds", "intra_phase_time", "optimal_time",
    "ratio_bound", "simulate_batch", "simulate_fast", "simulate_spreadout", "split_deliveries",
    "spreadout_completion_units", "spreadout_intra", "spreadout_stages", "stage_redistribution",
    "step_cost", "synthesize_spreadout",
]


@dataclass(frozen=True)
class Timeline:
    """Per-phase breakdown of a schedule's completion time (simulate.py:38-55).

    From simulate_fast / simulate_spreadout it is the modelled time; from
    FastComm.measured_timeline() the same fields are measured on the device.
    """

    t_balance: float
    t_intra_a2a: float
    scale_out: tuple[float, ...]
    redistribution: tuple[float, ...]
    total: float

    def to_json_dict(self) -> dict:
        return {"t_balance": self.t_balance, "t_intra_a2a": self.t_intra_a2a,
                "scale_out": list(self.scale_out), "redistribution": list(self.redistribution),
                "total": self.total}


@dataclass(frozen=True)
class BoundsReport:
    """Closed-form bounds for one instance (bounds.py:17-26)."""

    t_optimal: float
    t_fast_worstcase: float
    ratio_bound: float
    algo_bw: float
    assumption_ok: bool


@dataclass(frozen=True, eq=False)
class SpreadoutSchedule:
    """The shifted baseline: server totals plus its stages (pipeline.py:43-49)."""

    server: ServerMatrix
    gpus_per_server: int
    stages: tuple[PermutationStage, ...]


# ---------------------------------------------------------------- host scalars
def step_cost(nbytes: float, bw: float, t: Topology) -> float:
    """Wakeup plus transfer; zero bytes cost nothing (simulate.py:58-66)."""
    if bw <= 0:
        raise ValidationError("bandwidth must be positive")
    if nbytes < 0:
        raise ValidationError("byte count must be non-negative")
    if nbytes == 0:
        return 0.0
    return t.wakeup_delay + nbytes / bw


def intra_phase_time(moves: Iterable[IntraMove], t: Topology) -> float:
    """One batch of concurrent intra-server moves: the busiest GPU's send or
    receive total over scale-up (simulate.py:69-90)."""
    send: dict[tuple[int, int], int] = {}
    recv: dict[tuple[int, int], int] = {}
    for mv in moves:
        send[(mv.server, mv.from_gpu)] = send.get((mv.server, mv.from_gpu), 0) + mv.bytes
        recv[(mv.server, mv.to_gpu)] = recv.get((mv.server, mv.to_gpu), 0) + mv.bytes
    worst = max([0, *send.values(), *recv.values()])
    return step_cost(worst, t.scaleup_bw, t)


def ratio_bound(t: Topology) -> float:
    """Topology-only ceiling on worst-case / optimal (bounds.py:78-82)."""
    m, n = t.gpus_per_server, t.n_servers
    return 1.0 + (t.scaleout_bw / t.scaleup_bw) * (m + m / n)


def split_deliveries(table: np.ndarray, deliveries: Sequence[int]) -> list[np.ndarray]:
    """Per-stage pieces of a redistribution table: floor(cell * r_k / T) for
    all but the last delivery, which takes the remainder (balance.py:177-207).
    Exact for any magnitude (Python integers)."""
    total = int(np.asarray(table).sum())
    if sum(int(r) for r in deliveries) != total:
        raise ValidationError("stage deliveries must sum to the pair's tile total")
    table = np.asarray(table, dtype=np.int64)
    if total == 0:
        return [np.zeros_like(table) for _ in deliveries]
    cells = table.astype(object)
    pieces, acc = [], np.zeros(table.shape, dtype=object)
    for k, r in enumerate(deliveries):
        piece = cells - acc if k == len(deliveries) - 1 else cells * int(r) // total
        acc = acc + piece
        pieces.append(piece.astype(np.int64))
    return pieces


def stage_redistribution(plan: BalancePlan, stage_matching: Iterable[tuple[int, int]],
                         delivered: Mapping[tuple[int, int], int] | None = None,
                         earlier: Mapping[tuple[int, int], Sequence[int]] | None = None
                         ) -> list[IntraMove]:
    """Intra-server moves placing one stage's arrivals (balance.py:210-265)."""
    pairs = list(stage_matching)
    if len({i for i, _ in pairs}) != len(pairs) or len({j for _, j in pairs}) != len(pairs):
        raise ValidationError("stage matching must be one-to-one")
    moves: list[IntraMove] = []
    for i, j in pairs:
        if (i, j) not in plan.redistribution:
            raise ValidationError(f"unknown server pair ({i},{j})")
        table = plan.redistribution[(i, j)]
        total = int(table.sum())
        if total == 0:
            continue
        if delivered is None:
            piece = table
        else:
            r = int(delivered[(i, j)])
            prior = [int(x) for x in (earlier or {}).get((i, j), ())]
            done = sum(prior) + r
            if done > total:
                raise ValidationError(f"pair ({i},{j}) over-delivered: {done} > {total}")
            if done == total:
                piece = split_deliveries(table, prior + [r])[-1]
            else:
                piece = split_deliveries(table, [r, total - r])[0]
        m = table.shape[0]
        for p in range(m):
            for q in range(m):
                if p != q and piece[p, q] > 0:
                    moves.append(IntraMove(server=j, from_gpu=p, to_gpu=q, for_dst_server=j,
                                           bytes=int(piece[p, q])))
    return moves


def spreadout_intra(ops: np.ndarray, t: Topology, server: int = 0) -> list[list[IntraMove]]:
    """Shifted rounds for one server's internal all-to-all (spreadout.py:39-67)."""
    m = t.gpus_per_server
    ops = np.asarray(ops)
    if ops.shape != (m, m):
        raise ValidationError(f"intra tile must be {m}x{m}, got {ops.shape}")
    rounds = []
    for shift in range(1, m):
        rounds.append([IntraMove(server=server, from_gpu=g, to_gpu=(g + shift) % m,
                                 for_dst_server=server, bytes=int(ops[g, (g + shift) % m]))
                       for g in range(m) if int(ops[g, (g + shift) % m]) > 0])
    return rounds


# ------------------------------------------------------------- device model
def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_09764_b200 simulate needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _topo_struct(t: Topology) -> FastSimTopo:
    if t.scaleup_bw <= 0 or t.scaleout_bw <= 0:
        raise ValidationError("bandwidth must be positive")
    return FastSimTopo(float(t.scaleup_bw), float(t.scaleout_bw), float(t.wakeup_delay))


class SimBuffers:
    """Device outputs of fast_simulate_batch for B schedules."""

    def __init__(self, B: int, n: int, m: int, stage_stride: int, device=None):
        dev = device or _device()
        f64, i32, i64 = torch.float64, torch.int32, torch.int64
        e = lambda *shape, dt: torch.zeros(shape, dtype=dt, device=dev)  # noqa: E731
        K, N1 = max(stage_stride, 1), max(n - 1, 1)
        self.B, self.n, self.m, self.stage_stride = B, n, m, stage_stride
        self.t_balance, self.t_intra, self.total = e(B, dt=f64), e(B, dt=f64), e(B, dt=f64)
        self.scale_out, self.redistribution = e(B, K, dt=f64), e(B, K, dt=f64)
        self.t_optimal, self.t_worstcase = e(B, dt=f64), e(B, dt=f64)
        self.assumption_ok, self.status = e(B, dt=i32), e(B, dt=i32)
        self.so_weight = e(B, N1, dt=i64)
        self.so_server, self.so_demand = e(B, N1, dt=f64), e(B, N1, dt=f64)
        self.so_total = e(B, 2, dt=f64)
        ws = _lib.load().fast_sim_workspace_bytes(B, n, m, stage_stride)
        self.workspace = torch.empty(max(int(ws), 256), dtype=torch.uint8, device=dev)
        self.struct = FastSimOut(*(x.data_ptr() for x in (
            self.t_balance, self.t_intra, self.scale_out, self.redistribution, self.total,
            self.t_optimal, self.t_worstcase, self.assumption_ok, self.so_weight,
            self.so_server, self.so_demand, self.so_total, self.status, self.workspace)))


def _launch(inp: dict, B: int, n: int, m: int, t: Topology, out: SimBuffers,
            stream: torch.cuda.Stream | None = None) -> SimBuffers:
    ptr = lambda x: None if x is None else x.data_ptr()  # noqa: E731
    s_in = FastSimIn(*(ptr(inp.get(k)) for k in (
        "balanced", "server", "common_sum", "move_count", "moves", "n_stages", "stage_order",
        "stage_weight", "stage_perm", "stage_bytes", "status", "demand")),
        int(inp["move_slots"]), int(inp["stage_stride"]))
    topo = _topo_struct(t)
    sh = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    rc = _lib.load().fast_simulate_batch(ctypes.byref(s_in), B, n, m, ctypes.byref(topo),
                                         ctypes.byref(out.struct), sh)
    _lib.check_rc(rc, "fast_simulate_batch")
    out._inp = inp  # keep the inputs alive until the stream has consumed them
    return out


def simulate_batch(bufs, t: Topology, demand: torch.Tensor | None = None,
                   out: SimBuffers | None = None,
                   stream: torch.cuda.Stream | None = None) -> SimBuffers:
    """simulate_fast + simulate_spreadout + bounds for every schedule of a
    SynthBuffers batch, on the device (stream-ordered, no sync).  demand: the
    batch's original D [B, G, G] (enables the spreadout demand mode)."""
    from .synth import stage_cap

    n, m = bufs.n, bufs.m
    if (t.n_servers, t.gpus_per_server) != (n, m):
        raise ValidationError("plan and topology dimensions disagree")
    inp = dict(balanced=bufs.balanced, server=bufs.server, common_sum=bufs.common_sum,
               move_count=bufs.move_count, moves=bufs.moves, n_stages=bufs.n_stages,
               stage_order=bufs.stage_order, stage_weight=bufs.stage_weight,
               stage_perm=bufs.stage_perm, stage_bytes=bufs.stage_bytes, status=bufs.status,
               demand=None if demand is None else demand.contiguous(),
               move_slots=max(m - 1, 1), stage_stride=stage_cap(n))
    out = out or SimBuffers(bufs.B, n, m, stage_cap(n), bufs.balanced.device)
    return _launch(inp, bufs.B, n, m, t, out, stream)


def _raise(status: int) -> None:
    if status == _lib.FAST_EVALIDATION:
        raise ValidationError("stages must be sorted by ascending weight")
    if status != _lib.FAST_OK:
        raise InternalInvariantError(
            "stage bytes disagree with the redistribution tables, or the modelled "
            "completion fell below the scale-out lower bound")


def _tile_totals(sizes: np.ndarray, n: int, m: int) -> np.ndarray:
    return sizes.reshape(n, m, n, m).sum(axis=(1, 3)).astype(np.int64)


def _pack_objects(plan: BalancePlan, stages: Sequence[PermutationStage], t: Topology) -> dict:
    n, m = t.n_servers, t.gpus_per_server
    G = n * m
    re = np.asarray(plan.reshaped.sizes, dtype=np.int64)
    bal = np.zeros((G, G), np.int64)
    for i in range(n):
        bal[i * m:(i + 1) * m, i * m:(i + 1) * m] = re[i * m:(i + 1) * m, i * m:(i + 1) * m]
    for (i, j), table in plan.redistribution.items():
        if 0 <= i < n and 0 <= j < n and i != j:
            bal[i * m:(i + 1) * m, j * m:(j + 1) * m] = table
    srv = _tile_totals(re, n, m)
    T = n * (n - 1)
    per: list[list[IntraMove]] = [[] for _ in range(T)]
    for mv in plan.moves:
        i, j = mv.server, mv.for_dst_server
        if not (0 <= i < n and 0 <= j < n and i != j):
            raise ValidationError(f"intra move for unknown tile ({i},{j})")
        per[i * (n - 1) + (j if j < i else j - 1)].append(mv)
    slots = max([1, *map(len, per)])
    moves = np.zeros((T, slots, 2), np.int64)
    cnt = np.zeros(T, np.int32)
    for t_, lst in enumerate(per):
        cnt[t_] = len(lst)
        for u, mv in enumerate(lst):
            moves[t_, u, 0] = mv.bytes
            moves[t_, u, 1] = (int(mv.to_gpu) << 32) | (int(mv.from_gpu) & 0xFFFFFFFF)
    S = len(stages)
    K = max(S, 1)
    weight = np.zeros(K, np.int64)
    perm = np.zeros((K, n), np.uint8)
    sb = np.zeros((K, n), np.int64)
    for k, st in enumerate(stages):
        weight[k] = st.weight
        for src, dst, b in st.edges:
            if not 0 <= src < n:
                raise InternalInvariantError(f"stage edge for unknown server pair ({src},{dst})")
            perm[k, src] = dst if 0 <= dst < n else src  # src == dst: unknown pair
            sb[k, src] = b if b > 0 else -1
    dev = _device()
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    return dict(balanced=tt(bal), server=tt(srv), common_sum=tt(np.array([max_rc(ServerMatrix(srv))])),
                move_count=tt(cnt), moves=tt(moves), n_stages=tt(np.array([S], np.int32)),
                stage_order=tt(np.arange(K, dtype=np.int32)), stage_weight=tt(weight),
                stage_perm=tt(perm), stage_bytes=tt(sb), status=None, demand=None,
                move_slots=slots, stage_stride=K)


def _fetch(out: SimBuffers) -> dict:
    torch.cuda.current_stream().synchronize()
    return {k: getattr(out, k).cpu().numpy() for k in (
        "t_balance", "t_intra", "scale_out", "redistribution", "total", "t_optimal",
        "t_worstcase", "assumption_ok", "so_weight", "so_server", "so_demand", "so_total",
        "status")}


def simulate_fast(plan: BalancePlan, stages: Sequence[PermutationStage], t: Topology) -> Timeline:
    """Pipelined cost model of a balanced plan and its sorted stages
    (simulate.py:107-193), evaluated by the device kernel."""
    n, m = t.n_servers, t.gpus_per_server
    if (plan.reshaped.n_servers, plan.reshaped.gpus_per_server) != (n, m):
        raise ValidationError("plan and topology dimensions disagree")
    stages = list(stages)
    inp = _pack_objects(plan, stages, t)
    out = _fetch(_launch(inp, 1, n, m, t, SimBuffers(1, n, m, inp["stage_stride"])))
    _raise(int(out["status"][0]))
    S = len(stages)
    return Timeline(t_balance=float(out["t_balance"][0]), t_intra_a2a=float(out["t_intra"][0]),
                    scale_out=tuple(float(x) for x in out["scale_out"][0][:S]),
                    redistribution=tuple(float(x) for x in out["redistribution"][0][:S]),
                    total=float(out["total"][0]))


def _server_only(s: ServerMatrix, t: Topology, demand: DemandMatrix | None) -> dict:
    """Model outputs that depend only on a server matrix (+ optional demand):
    the kernel with zero stages and empty tables."""
    n, m = s.n_servers, t.gpus_per_server
    G = n * m
    dev = _device()
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    T = max(n * (n - 1), 1)
    inp = dict(balanced=torch.zeros((G, G), dtype=torch.int64, device=dev),
               server=tt(np.asarray(s.totals, dtype=np.int64)),
               common_sum=tt(np.array([max_rc(s)], np.int64)),
               move_count=torch.zeros(T, dtype=torch.int32, device=dev),
               moves=torch.zeros((T, 1, 2), dtype=torch.int64, device=dev),
               n_stages=torch.zeros(1, dtype=torch.int32, device=dev),
               stage_order=torch.zeros(1, dtype=torch.int32, device=dev),
               stage_weight=torch.zeros(1, dtype=torch.int64, device=dev),
               stage_perm=torch.zeros((1, n), dtype=torch.uint8, device=dev),
               stage_bytes=torch.zeros((1, n), dtype=torch.int64, device=dev), status=None,
               demand=None if demand is None else tt(np.asarray(demand.sizes, np.int64)),
               move_slots=1, stage_stride=1)
    topo = Topology(n, m, t.scaleup_bw, t.scaleout_bw, t.wakeup_delay)
    return _fetch(_launch(inp, 1, n, m, topo, SimBuffers(1, n, m, 1)))


def simulate_spreadout(s: ServerMatrix, t: Topology,
                       demand: DemandMatrix | None = None) -> Timeline:
    """The shifted baseline's cost: stage durations add up (simulate.py:196-242)."""
    n, m = s.n_servers, t.gpus_per_server
    if n != t.n_servers:
        raise ValidationError("server matrix and topology dimensions disagree")
    if demand is not None and (demand.n_servers, demand.gpus_per_server) != (n, m):
        raise ValidationError("demand matrix and topology dimensions disagree")
    out = _server_only(s, t, demand)
    dur = out["so_server" if demand is None else "so_demand"][0][: n - 1]
    total = out["so_total"][0][0 if demand is None else 1]
    return Timeline(t_balance=0.0, t_intra_a2a=0.0, scale_out=tuple(float(x) for x in dur),
                    redistribution=tuple(0.0 for _ in dur), total=float(total))


def spreadout_stages(s: ServerMatrix) -> list[PermutationStage]:
    """The n-1 shifted stages; weight = largest edge (spreadout.py:19-31)."""
    n = s.n_servers
    t = Topology(n, 1)
    w = _server_only(s, t, None)["so_weight"][0]
    off = s.off_diagonal()
    from .schedule import _fast_stage

    out = []
    for shift in range(1, n):
        edges = tuple(sorted((src, (src + shift) % n, int(off[src, (src + shift) % n]))
                             for src in range(n)))
        out.append(_fast_stage(int(w[shift - 1]), edges))
    return out


def spreadout_completion_units(s: ServerMatrix) -> int:
    """Sum of per-stage maxima in bytes (spreadout.py:34-36)."""
    return sum(st.weight for st in spreadout_stages(s))


def synthesize_spreadout(d: DemandMatrix, t: Topology) -> SpreadoutSchedule:
    """Reduce to server level and emit the shifted stages (pipeline.py:62-69)."""
    server = reduce_to_server_level(d, t)
    return SpreadoutSchedule(server=server, gpus_per_server=t.gpus_per_server,
                             stages=tuple(spreadout_stages(server)))


def _warn(ok: bool) -> bool:
    if not ok:
        warnings.warn("some server's intra traffic exceeds its average cross-server demand; "
                      "the bound assumes it hides behind scale-out transfers", stacklevel=3)
    return ok


def intra_assumption_holds(s: ServerMatrix) -> bool:
    """S_i <= (1/n) sum_j T_ij for every server (bounds.py:27-35)."""
    return bool(_server_only(s, Topology(s.n_servers, 1), None)["assumption_ok"][0])


def optimal_time(s: ServerMatrix, t: Topology) -> float:
    """Scale-out lower bound max_rc / (m B2) (bounds.py:49-57)."""
    out = _server_only(s, t, None)
    _warn(bool(out["assumption_ok"][0]))
    return float(out["t_optimal"][0])


def fast_worstcase_time(s: ServerMatrix, t: Topology) -> float:
    """Balancing + staging + redistribution ceilings (bounds.py:60-75)."""
    out = _server_only(s, t, None)
    _warn(bool(out["assumption_ok"][0]))
    return float(out["t_worstcase"][0])


def bounds_report(s: ServerMatrix, t: Topology, total_bytes: int,
                  completion_s: float) -> BoundsReport:
    """All bounds plus the achieved algorithmic bandwidth (bounds.py:101-120)."""
    from . import algorithmic_bandwidth

    out = _server_only(s, t, None)
    ok = _warn(bool(out["assumption_ok"][0]))
    return BoundsReport(t_optimal=float(out["t_optimal"][0]),
                        t_fast_worstcase=float(out["t_worstcase"][0]), ratio_bound=ratio_bound(t),
                        algo_bw=algorithmic_bandwidth(total_bytes, s.n_servers * t.gpus_per_server,
                                                      completion_s),
                        assumption_ok=ok)
