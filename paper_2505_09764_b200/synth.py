"""GPU schedule synthesis behind tiersched's scheduler API.

Drop-in entry points (same names, arguments and error classes as the
reference):

    synthesize_fast(d, t) -> Schedule                 pipeline.py:52
    build_balance_plan(d, t) -> BalancePlan           balance.py:139
    decompose_server_matrix(s) -> Decomposition       birkhoff.py:269
    embed_doubly_stochastic(s) -> (embedded, aux)     birkhoff.py:75
    decompose(embedded) -> list[PermutationStage]     birkhoff.py:140

plus the batched device API used by the executor and the benchmarks:

    synthesize_packed(D, n, m) -> SynthBuffers  (D: cuda int64 [B,G,G])

Every call runs the sm_100a kernels in libfastb200.so on the current CUDA
stream.  There is no CPU fallback: without a CUDA device these raise.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .model import (DemandMatrix, InternalInvariantError, ServerMatrix, TileView, Topology,
                    ValidationError)
from .schedule import (MOVE_DTYPE, STRIP_DTYPE, BalancePlan, Decomposition, IntraMove,
                       PackedSchedule, PermutationStage, Schedule, _fast_stage,
                       balanced_from_compact, stage_bytes_from_strip)

FAST_MAX_SERVERS = 128  # include/fastb200.h


def stage_cap(n: int) -> int:
    return n * n - 2 * n + 2


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_09764_b200 synthesis needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream_handle(stream: torch.cuda.Stream | None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class SynthBuffers:
    """Device-resident packed schedules for a batch (fast_sched_bufs).

    stage_bytes=False skips the per-edge [B, K, n] real-byte array (the
    decomposition then only records the aux run-out table, `strip`, from which
    the host rebuilds it); compact=True adds the strip table and the changed-
    cell masks of the balanced cross tiles (fast_compact_batch input)."""

    def __init__(self, B: int, n: int, m: int, device: torch.device | None = None,
                 with_balance: bool = True, stage_bytes: bool = True, compact: bool = False):
        dev = device or _device()
        G, T, S, K = n * m, n * (n - 1), max(m - 1, 1), stage_cap(n)
        self.B, self.n, self.m = B, n, m
        i64, i32, u8 = torch.int64, torch.int32, torch.uint8
        e = lambda *shape, dt: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
        gb = G if with_balance else 1
        self.balanced = e(B, gb, gb, dt=i64)
        self.server = e(B, n, n, dt=i64)
        self.move_count = e(B, T, dt=i32)
        self.moves = e(B, T, S, 2, dt=i64)  # fast_move is 16 bytes
        self.common_sum = e(B, dt=i64)
        self.aux = e(B, n, n, dt=i64)
        self.n_raw = e(B, dt=i32)
        self.stage_weight = e(B, K, dt=i64)
        self.stage_perm = e(B, K, n, dt=u8)
        self.stage_bytes = e(B, K, n, dt=i64) if stage_bytes or not compact else None
        self.n_stages = e(B, dt=i32)
        self.stage_order = e(B, K, dt=i32)
        self.status = e(B, dt=i32)
        ws = _lib.load().fast_synth_workspace_bytes(B, n)
        self.workspace = e(max(int(ws), 16), dt=u8)
        self.strip = e(B, 2 * n + 2, 2, dt=i64) if compact else None  # fast_strip_rec: 16 B
        self.tile_mask = e(B, max(T, 1), dt=i64) if compact and m <= 8 else None
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        self._struct = _lib.FastSchedBufs(*(ptr(t) for t in (
            self.balanced, self.server, self.move_count, self.moves, self.common_sum,
            self.aux, self.n_raw, self.stage_weight, self.stage_perm, self.stage_bytes,
            self.n_stages, self.stage_order, self.status, self.workspace, self.strip,
            self.tile_mask)))

    @property
    def struct(self) -> _lib.FastSchedBufs:
        return self._struct

    def output_nbytes(self) -> int:
        """Bytes of the packed schedule (what a D2H of the result moves)."""
        ts = (self.balanced, self.server, self.move_count, self.moves, self.common_sum,
              self.aux, self.n_raw, self.stage_weight, self.stage_perm, self.stage_bytes,
              self.n_stages, self.stage_order, self.status)
        return sum(t.numel() * t.element_size() for t in ts if t is not None)

    def host(self, b: int | None = None) -> list[PackedSchedule]:
        """Copy to host and split per matrix (synchronizes)."""
        h = {k: getattr(self, k).cpu().numpy() for k in (
            "balanced", "server", "move_count", "moves", "common_sum", "aux", "n_raw",
            "stage_weight", "stage_perm", "n_stages", "stage_order", "status")}
        h["stage_bytes"] = None if self.stage_bytes is None else self.stage_bytes.cpu().numpy()
        strip = None if self.strip is None else self.strip.cpu().numpy().view(STRIP_DTYPE)
        moves = h["moves"].view(MOVE_DTYPE).reshape(h["moves"].shape[:3])
        idx = range(self.B) if b is None else [b]
        out = []
        for i in idx:
            k, s = int(h["n_raw"][i]), int(h["n_stages"][i])
            if h["stage_bytes"] is not None:
                sb = h["stage_bytes"][i][:k]
            else:
                sb = stage_bytes_from_strip(h["stage_weight"][i][:k], h["stage_perm"][i][:k],
                                            strip[i].reshape(-1))
            out.append(PackedSchedule(
                n=self.n, m=self.m, status=int(h["status"][i]), balanced=h["balanced"][i],
                server=h["server"][i], move_count=h["move_count"][i], moves=moves[i],
                common_sum=int(h["common_sum"][i]), aux=h["aux"][i], n_raw=k,
                stage_weight=h["stage_weight"][i][:k], stage_perm=h["stage_perm"][i][:k],
                stage_bytes=sb, n_stages=s,
                stage_order=h["stage_order"][i][:s]))
        return out


def synthesize_packed(D: torch.Tensor, n: int, m: int, bufs: SynthBuffers | None = None,
                      stream: torch.cuda.Stream | None = None) -> SynthBuffers:
    """Batched synthesize_fast on the device (stream-ordered, no sync).

    D: cuda int64 [B, n*m, n*m].  Per-matrix status lands in bufs.status.
    """
    if D.dtype != torch.int64 or not D.is_cuda or D.dim() != 3:
        raise ValidationError("D must be a cuda int64 tensor [B, G, G]")
    B = D.shape[0]
    if D.shape[1:] != (n * m, n * m):
        raise ValidationError(f"D shape {tuple(D.shape)} does not match n={n}, m={m}")
    D = D.contiguous()
    if bufs is None:
        bufs = SynthBuffers(B, n, m, D.device)
    rc = _lib.load().fast_synth_batch(ctypes.c_void_p(D.data_ptr()), B, n, m,
                                      ctypes.byref(bufs.struct), _stream_handle(stream))
    _lib.check_rc(rc, "fast_synth_batch")
    return bufs


def _raise_status(code: int, what: str) -> None:
    if code == _lib.FAST_EVALIDATION:
        raise ValidationError(f"{what}: invalid input")
    if code != _lib.FAST_OK:
        raise InternalInvariantError(f"{what}: internal invariant broken (status {code})")


def _demand_batch(ds: Sequence[DemandMatrix] | np.ndarray, t: Topology) -> np.ndarray:
    if isinstance(ds, np.ndarray):
        return np.ascontiguousarray(ds, dtype=np.int64)
    for d in ds:
        if (d.n_servers, d.gpus_per_server) != (t.n_servers, t.gpus_per_server):
            raise ValidationError(
                f"matrix is {d.n_servers}x{d.gpus_per_server} but topology is "
                f"{t.n_servers}x{t.gpus_per_server}")
    return np.stack([d.sizes for d in ds]).astype(np.int64, copy=False)


def synthesize_fast_batch(ds: Sequence[DemandMatrix] | np.ndarray, t: Topology) -> list[Schedule]:
    """synthesize_fast over many matrices in one set of kernel launches."""
    n, m = t.n_servers, t.gpus_per_server
    D = torch.from_numpy(_demand_batch(ds, t)).to(_device())
    packed = synthesize_packed(D, n, m).host()
    out = []
    for p in packed:
        _raise_status(p.status, "synthesize_fast")
        out.append(p.to_schedule())
    return out


def synthesize_fast(d: DemandMatrix, t: Topology) -> Schedule:
    """Balance, reduce, decompose, strip, sort -- on the GPU (pipeline.py:52)."""
    return synthesize_fast_batch([d], t)[0]


def build_balance_plan(d: DemandMatrix, t: Topology) -> BalancePlan:
    """Phase 1 only (balance.py:139-174), on the GPU."""
    n, m = t.n_servers, t.gpus_per_server
    D = torch.from_numpy(_demand_batch([d], t)).to(_device())
    bufs = SynthBuffers(1, n, m, D.device)
    rc = _lib.load().fast_balance_batch(ctypes.c_void_p(D.data_ptr()), 1, n, m,
                                        ctypes.byref(bufs.struct), _stream_handle(None))
    _lib.check_rc(rc, "fast_balance_batch")
    st = int(bufs.status.cpu()[0])
    _raise_status(st, "build_balance_plan")
    h = {k: getattr(bufs, k)[0].cpu().numpy() for k in ("balanced", "server", "move_count", "moves")}
    p = PackedSchedule(n=n, m=m, status=st, balanced=h["balanced"], server=h["server"],
                       move_count=h["move_count"],
                       moves=h["moves"].view(MOVE_DTYPE).reshape(h["moves"].shape[:2]),
                       common_sum=0, aux=np.zeros((n, n), np.int64), n_raw=0,
                       stage_weight=np.zeros(0, np.int64), stage_perm=np.zeros((0, n), np.uint8),
                       stage_bytes=np.zeros((0, n), np.int64), n_stages=0,
                       stage_order=np.zeros(0, np.int32))
    return p.balance_plan()


def _decompose_packed(S: np.ndarray, mode: int) -> PackedSchedule:
    S = np.ascontiguousarray(S, dtype=np.int64)
    n = S.shape[0]
    if S.ndim != 2 or S.shape[1] != n:
        raise ValidationError("decompose expects a square matrix")
    dev = _device()
    St = torch.from_numpy(S[None].copy()).to(dev)
    bufs = SynthBuffers(1, n, 1, dev, with_balance=False)
    rc = _lib.load().fast_decompose_batch(ctypes.c_void_p(St.data_ptr()), 1, n, mode,
                                          ctypes.byref(bufs.struct), _stream_handle(None))
    _lib.check_rc(rc, "fast_decompose_batch")
    return bufs.host(0)[0]


def decompose_server_matrix(s: ServerMatrix) -> Decomposition:
    """Embed + decompose a server matrix (birkhoff.py:269-280), on the GPU."""
    p = _decompose_packed(s.totals, _lib.FAST_DEC_SERVER)
    _raise_status(p.status, "decompose_server_matrix")
    return p.decomposition()


def embed_doubly_stochastic(s: ServerMatrix) -> tuple[np.ndarray, np.ndarray]:
    """Northwest-corner embedding (birkhoff.py:75-108), on the GPU."""
    p = _decompose_packed(s.totals, _lib.FAST_DEC_SERVER)
    _raise_status(p.status, "embed_doubly_stochastic")
    return s.off_diagonal() + p.aux, p.aux.copy()


def decompose(embedded: np.ndarray) -> list[PermutationStage]:
    """Birkhoff peeling of a doubly stochastic matrix (birkhoff.py:140-222)."""
    e = np.asarray(embedded)
    if e.ndim != 2 or e.shape[0] != e.shape[1]:
        raise ValidationError("decompose expects a square matrix")
    if not np.issubdtype(e.dtype, np.integer):
        raise ValidationError("decompose expects an integer matrix")
    # the reference's remaining checks, with its messages (birkhoff.py:155-163);
    # the kernel checks the same on the device (status 2)
    if np.any(e < 0):
        raise ValidationError("decompose expects non-negative entries")
    rows, cols = e.sum(axis=1), e.sum(axis=0)
    if e.size and not (np.all(rows == rows[0]) and np.all(cols == rows[0])):
        raise ValidationError("decompose expects equal row and column sums")
    p = _decompose_packed(e.astype(np.int64), _lib.FAST_DEC_DOUBLY_STOCHASTIC)
    _raise_status(p.status, "decompose")
    return list(p.raw_stages())


# fixed-size fields of the compact host result, copied whole per chunk
_COMPACT_FIELDS = ("server", "move_count", "moves", "common_sum", "aux", "n_raw",
                   "stage_weight", "stage_perm", "n_stages", "stage_order", "status", "strip",
                   "tile_mask")
# m > 8 (no 64-bit changed-cell mask per tile): the balanced matrix itself
_WIDE_FIELDS = _COMPACT_FIELDS[:-1] + ("balanced",)


def _host_fields(m: int) -> tuple:
    return _COMPACT_FIELDS if m <= 8 else _WIDE_FIELDS


class HostSchedules:
    """Compact pinned-host result of synthesize_host_batch for a batch.

    What crosses PCIe per matrix (config 5, n = 128, m = 8: ~5.9 MB instead
    of the 37.7 MB full device layout): the server matrix, moves, aux, the
    raw stage weights and permutations, the sort order, the aux run-out table
    (`strip`, replaces the [K, n] stage_bytes array) and the balanced cross
    tiles as changed-cell masks + values (`tile_mask`, `vals`; replaces the
    G x G balanced matrix, which is D outside those cells).  ``packed(b, D)``
    decodes one matrix into the full PackedSchedule (and thus the reference
    dataclasses / canonical JSON).  For m > 8 the G x G balanced matrix
    itself is copied instead of the masks and values."""

    def __init__(self, B: int, n: int, m: int, vals_capacity: int | None = None):
        G, T, S, K = n * m, n * (n - 1), max(m - 1, 1), stage_cap(n)
        shapes = {"server": ((B, n, n), torch.int64),
                  "move_count": ((B, T), torch.int32), "moves": ((B, T, S, 2), torch.int64),
                  "common_sum": ((B,), torch.int64), "aux": ((B, n, n), torch.int64),
                  "n_raw": ((B,), torch.int32), "stage_weight": ((B, K), torch.int64),
                  "stage_perm": ((B, K, n), torch.uint8), "n_stages": ((B,), torch.int32),
                  "stage_order": ((B, K), torch.int32), "status": ((B,), torch.int32),
                  "strip": ((B, 2 * n + 2, 2), torch.int64),
                  "tile_mask": ((B, max(T, 1)), torch.int64), "balanced": ((B, G, G), torch.int64)}
        shapes = {k: shapes[k] for k in _host_fields(m)}
        self.fields = _host_fields(m)
        self.B, self.n, self.m = B, n, m
        for k, (shape, dt) in shapes.items():
            setattr(self, k, torch.empty(shape, dtype=dt, pin_memory=True))
        self.val_base = torch.zeros(B + 1, dtype=torch.int64)
        self.vals = torch.empty(int(vals_capacity or B * max(T, 1) * 16), dtype=torch.int64,
                                pin_memory=True)
        self.n_vals = 0

    def fixed_nbytes(self) -> int:
        return sum(getattr(self, k).numel() * getattr(self, k).element_size()
                   for k in self.fields)

    def nbytes(self) -> int:
        """Bytes copied device -> host by the last synthesize_host_batch."""
        return self.fixed_nbytes() + 8 * self.n_vals + 8 * (self.B + 1)

    def packed(self, b: int, D: np.ndarray) -> PackedSchedule:
        """Decode matrix b (D: its host demand matrix) into the full layout."""
        n, m = self.n, self.m
        k, s = int(self.n_raw[b]), int(self.n_stages[b])
        w = self.stage_weight[b, :k].numpy()
        perm = self.stage_perm[b, :k].numpy()
        strip = self.strip[b].numpy().view(STRIP_DTYPE).reshape(-1)
        v0, v1 = int(self.val_base[b]), int(self.val_base[b + 1])
        st = int(self.status[b])
        if m > 8:
            bal = self.balanced[b].numpy() if st == 0 else np.array(D, dtype=np.int64)
        else:
            bal = (balanced_from_compact(D, self.tile_mask[b].numpy().view(np.uint64),
                                         self.vals[v0:v1].numpy(), n, m)
                   if st == 0 else np.array(D, dtype=np.int64))
        moves = self.moves[b].numpy().view(MOVE_DTYPE).reshape(self.moves.shape[1:3])
        return PackedSchedule(
            n=n, m=m, status=st, balanced=bal, server=self.server[b].numpy(),
            move_count=self.move_count[b].numpy(), moves=moves,
            common_sum=int(self.common_sum[b]), aux=self.aux[b].numpy(), n_raw=k,
            stage_weight=w, stage_perm=perm, stage_bytes=stage_bytes_from_strip(w, perm, strip),
            n_stages=s, stage_order=self.stage_order[b, :s].numpy())


class HostSynthPipeline:
    """synthesize_fast over batches held in (pinned) HOST memory, producing
    the compact host result (HostSchedules) -- the e2e path.

    A batch is split into chunks; each chunk has its own stream and device
    buffers: its H2D, synthesis (+ fast_compact_batch) and the D2H of its
    fixed-size fields are stream-ordered, and the chunks are independent, so
    the copy engines stream inputs and results while every chunk's
    (latency-bound) decomposition runs on the SMs.  The variable-length
    changed-cell values of a chunk are copied once its count has landed on
    the host.

    `depth` buffer sets rotate between consecutive batches: ``submit`` only
    enqueues (returning a ticket) and ``result`` completes a ticket, so a
    caller streaming batches keeps the next batch's H2D and kernels in flight
    while the previous batch's chain tail and D2H finish (``run``)."""

    def __init__(self, B: int, n: int, m: int, chunk: int = 125, depth: int = 2, device=None):
        dev = device or _device()
        lib = _lib.load()
        self.B, self.n, self.m, self.dev = B, n, m, dev
        C = max(1, min(chunk, B))
        self.starts = list(range(0, B, C))
        sizes = [min(C, B - b0) for b0 in self.starts]
        T = n * (n - 1)
        self.sets = []
        for _ in range(max(1, depth)):
            self.sets.append(dict(
                bufs=[SynthBuffers(nb, n, m, dev, compact=True) for nb in sizes],
                dins=[torch.empty((nb, n * m, n * m), dtype=torch.int64, device=dev)
                      for nb in sizes],
                vals=[torch.empty(nb * max(T, 1) * m * m if m <= 8 else 1, dtype=torch.int64,
                                  device=dev) for nb in sizes],
                base=[torch.empty(nb + 1, dtype=torch.int64, device=dev) for nb in sizes],
                base_h=[torch.empty(nb + 1, dtype=torch.int64, pin_memory=True) for nb in sizes],
                ws=[torch.empty(int(lib.fast_compact_workspace_bytes(nb)), dtype=torch.uint8,
                                device=dev) for nb in sizes],
                streams=[torch.cuda.Stream(dev) for _ in sizes],
                events=[torch.cuda.Event() for _ in sizes]))
        self._next = 0

    def submit(self, D_host: torch.Tensor, out: HostSchedules, trace: list | None = None):
        """Enqueue one batch (no host synchronisation); returns a ticket."""
        n, m = self.n, self.m
        if (D_host.device.type != "cpu" or D_host.dtype != torch.int64 or D_host.dim() != 3
                or D_host.shape[0] != self.B):
            raise ValidationError(f"D_host must be a CPU int64 tensor [{self.B}, G, G]")
        lib = _lib.load()
        c = self.sets[self._next]
        self._next = (self._next + 1) % len(self.sets)
        cur = torch.cuda.current_stream(self.dev)
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if trace is not None else None
        if trace is not None:
            t_start = ev()
            t_start.record(cur)
            trace.append(t_start)
        for i, b0 in enumerate(self.starts):
            st, nb, bufs = c["streams"][i], c["dins"][i].shape[0], c["bufs"][i]
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                c["dins"][i].copy_(D_host[b0:b0 + nb], non_blocking=True)
                if trace is not None:
                    trace.append(("h2d", i, ev()))
                    trace[-1][2].record(st)
                sh = ctypes.c_void_p(st.cuda_stream)
                evs = None
                if trace is not None:
                    kev = [ev() for _ in range(4)]
                    trace.extend([("bal0", i, kev[0]), ("bal1", i, kev[1]), ("dec1", i, kev[2]),
                                  ("sort1", i, kev[3])])
                    for e in kev:
                        e.record(st)  # materialise
                    evs = (ctypes.c_void_p * 4)(*[e.cuda_event for e in kev])
                _lib.check_rc(lib.fast_synth_batch_ev(ctypes.c_void_p(c["dins"][i].data_ptr()),
                                                      nb, n, m, ctypes.byref(bufs.struct), sh,
                                                      evs), "fast_synth_batch")
                if m <= 8:
                    _lib.check_rc(lib.fast_compact_batch(
                        ctypes.byref(bufs.struct), nb, n, m,
                        ctypes.c_void_p(c["vals"][i].data_ptr()),
                        ctypes.c_void_p(c["base"][i].data_ptr()),
                        ctypes.c_void_p(c["ws"][i].data_ptr()), sh), "fast_compact_batch")
                else:  # no masks: no changed-cell values either
                    c["base"][i].zero_()
                if trace is not None:
                    trace.append(("synth", i, ev()))
                    trace[-1][2].record(st)
                c["base_h"][i].copy_(c["base"][i], non_blocking=True)
                c["events"][i].record(st)
                for f in out.fields:
                    getattr(out, f)[b0:b0 + nb].copy_(getattr(bufs, f), non_blocking=True)
                if trace is not None:
                    trace.append(("d2h", i, ev()))
                    trace[-1][2].record(st)
        return (c, out)

    def result(self, ticket, sync: bool = True) -> HostSchedules:
        """Complete a ticket: as each chunk's value count lands, enqueue the
        D2H of its changed-cell values; sync=True waits for the last copy."""
        c, out = ticket
        off = 0
        for i, b0 in enumerate(self.starts):
            c["events"][i].synchronize()
            nb = c["dins"][i].shape[0]
            base = c["base_h"][i]
            tot = int(base[nb])
            if off + tot > out.vals.numel():  # grow (first call at this size)
                for st in c["streams"]:
                    st.synchronize()
                grown = torch.empty(max(2 * out.vals.numel(), off + tot), dtype=torch.int64,
                                    pin_memory=True)
                grown[:off].copy_(out.vals[:off])
                out.vals = grown
            with torch.cuda.stream(c["streams"][i]):
                if tot:
                    out.vals[off:off + tot].copy_(c["vals"][i][:tot], non_blocking=True)
            out.val_base[b0:b0 + nb] = base[:nb] + off
            off += tot
        out.val_base[self.B] = off
        out.n_vals = off
        if sync:
            for st in c["streams"]:
                st.synchronize()
        return out

    def run(self, batches, outs) -> list[HostSchedules]:
        """Stream batches through the pipeline: up to `depth` batches are
        enqueued before the oldest is completed.  outs[t] receives batch t
        (rotate `depth` objects for a steady stream)."""
        pending, done = [], []
        for D_host, out in zip(batches, outs):
            pending.append(self.submit(D_host, out))
            if len(pending) >= len(self.sets):
                done.append(self.result(pending.pop(0)))
        while pending:
            done.append(self.result(pending.pop(0)))
        return done


def synthesize_host_batch(D_host: torch.Tensor, n: int, m: int, out: HostSchedules | None = None,
                          chunk: int = 125, device=None, _cache: dict = {},
                          trace: list | None = None) -> HostSchedules:
    """synthesize_fast over one batch in (pinned) HOST memory, synchronously
    (HostSynthPipeline with one buffer set, cached across calls)."""
    dev = device or _device()
    if D_host.device.type != "cpu" or D_host.dtype != torch.int64 or D_host.dim() != 3:
        raise ValidationError("D_host must be a CPU int64 tensor [B, G, G]")
    B = D_host.shape[0]
    out = out or HostSchedules(B, n, m)
    key = (str(dev), B, n, m, max(1, min(chunk, B)))
    if key not in _cache:  # device buffers and streams are reused across calls
        _cache.clear()
        _cache[key] = HostSynthPipeline(B, n, m, chunk, depth=1, device=dev)
    pipe = _cache[key]
    return pipe.result(pipe.submit(D_host, out, trace))


# ---------------------------------------------------------------------------
# Stage-level building blocks of the reference's balance / Birkhoff modules
# as standalone calls (the batched synthesis fuses them).
def balance_senders(tv: TileView) -> tuple[np.ndarray, list[IntraMove]]:
    """Equalize one cross tile's row sums (balance.py:77-126): the balance
    kernel on a two-server embedding of the tile."""
    if tv.is_intra:
        raise ValidationError("balance_senders expects a cross-server tile")
    e = np.asarray(tv.entries, dtype=np.int64)
    m = e.shape[0]
    if e.ndim != 2 or e.shape != (m, m):
        raise ValidationError("tile must be square")
    D = np.zeros((2 * m, 2 * m), np.int64)
    D[:m, m:] = e
    dev = _device()
    Dt = torch.from_numpy(D[None].copy()).to(dev)
    bufs = SynthBuffers(1, 2, m, dev)
    rc = _lib.load().fast_balance_batch(ctypes.c_void_p(Dt.data_ptr()), 1, 2, m,
                                        ctypes.byref(bufs.struct), _stream_handle(None))
    _lib.check_rc(rc, "fast_balance_batch")
    _raise_status(int(bufs.status.cpu()[0]), "balance_senders")
    bal = bufs.balanced[0, :m, m:].cpu().numpy().copy()
    cnt = int(bufs.move_count[0, 0].item())
    mv = bufs.moves[0, 0, :cnt].cpu().numpy().view(MOVE_DTYPE).reshape(-1)
    moves = [IntraMove(server=tv.src_server, from_gpu=int(x["from_gpu"]), to_gpu=int(x["to_gpu"]),
                       for_dst_server=tv.dst_server, bytes=int(x["bytes"])) for x in mv]
    return bal, moves


def merge_peer(balanced_tile: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """diag(row sums) plus the redistribution table (balance.py:129-136)."""
    rows = np.asarray(balanced_tile).sum(axis=1)
    if rows.size and int(rows.max() - rows.min()) > 1:
        raise ValidationError("merge_peer expects row sums differing by <= 1")
    return np.diag(rows).astype(np.int64), np.asarray(balanced_tile).astype(np.int64, copy=True)


def find_perfect_matching(support: np.ndarray) -> dict[int, int]:
    """Deterministic perfect matching (birkhoff.py:111-137): the
    decomposition's warp DFS (fast_match_batch)."""
    sp = np.asarray(support)
    if sp.ndim != 2 or sp.shape[0] != sp.shape[1]:
        raise ValidationError("support must be a square matrix")
    n = sp.shape[0]
    if n == 0:
        return {}
    if n > FAST_MAX_SERVERS:
        raise ValidationError(f"support larger than {FAST_MAX_SERVERS} rows")
    dev = _device()
    st = torch.from_numpy((sp != 0).astype(np.uint8)[None].copy()).to(dev)
    rm = torch.empty((1, n), dtype=torch.int32, device=dev)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    rc = _lib.load().fast_match_batch(ctypes.c_void_p(st.data_ptr()), 1, n,
                                      ctypes.c_void_p(rm.data_ptr()),
                                      ctypes.c_void_p(status.data_ptr()), _stream_handle(None))
    _lib.check_rc(rc, "fast_match_batch")
    if int(status.item()) != _lib.FAST_OK:
        raise InternalInvariantError("support matrix has no perfect matching")
    r = rm[0].cpu().numpy()
    return {u: int(r[u]) for u in range(n)}


def _strip_sort(stages: Sequence[PermutationStage], aux: np.ndarray | None, mode: int):
    stages = list(stages)
    K = len(stages)
    n = 1
    for st in stages:
        for s, d, _ in st.edges:
            n = max(n, int(s) + 1, int(d) + 1)
    if aux is not None:
        aux = np.asarray(aux, dtype=np.int64)
        n = max(n, aux.shape[0])
    Kc = max(K, 1)
    w = np.zeros(Kc, np.int64)
    dst = np.full((Kc, n), -1, np.int16)
    b = np.zeros((Kc, n), np.int64)
    for k, st in enumerate(stages):
        w[k] = st.weight
        for s, d, x in st.edges:
            dst[k, s], b[k, s] = d, x
    A = np.zeros((n, n), np.int64)
    if aux is not None:
        A[: aux.shape[0], : aux.shape[1]] = aux
    dev = _device()
    tt = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    wt, dt, bt, at = tt(w), tt(dst), tt(b), tt(A)
    order = torch.empty(Kc, dtype=torch.int32, device=dev)
    real = torch.empty((Kc, n), dtype=torch.int64, device=dev)
    n_out = torch.zeros(1, dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    ws = torch.empty(int(lib.fast_strip_sort_workspace_bytes(K, n)), dtype=torch.uint8,
                     device=dev)
    P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
    rc = lib.fast_strip_sort(P(wt), P(dt), P(bt), P(at), K, n, mode, P(order), P(real), P(n_out),
                             P(status), P(ws), _stream_handle(None))
    _lib.check_rc(rc, "fast_strip_sort")
    st = int(status.item())
    if st != _lib.FAST_OK:
        raise InternalInvariantError("auxiliary bytes left unconsumed")
    k_out = int(n_out.item())
    return stages, order[:k_out].cpu().numpy(), real.cpu().numpy(), dst


def strip_auxiliary(stages: Sequence[PermutationStage], aux: np.ndarray) -> list[PermutationStage]:
    """Charge the auxiliary padding greedily, drop emptied edges and stages
    (birkhoff.py:225-252), on the device (fast_strip_sort)."""
    stages, order, real, dst = _strip_sort(stages, aux, 1)
    out = []
    for k in order:
        edges = tuple((u, int(dst[k, u]), int(real[k, u])) for u in range(dst.shape[1])
                      if dst[k, u] >= 0 and real[k, u] > 0)
        out.append(_fast_stage(stages[k].weight, edges))
    return out


def sort_stages_ascending(stages: Sequence[PermutationStage]) -> list[PermutationStage]:
    """Stable sort by (weight, first (src, dst) edge) (birkhoff.py:255-266),
    on the device (fast_strip_sort)."""
    stages, order, _, _ = _strip_sort(stages, None, 2)
    return [stages[int(k)] for k in order]
