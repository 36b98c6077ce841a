"""FAST alltoallv execution over NVSwitch -- the executor the reference only
models (tiersched.simulate_fast, simulate.py:107-193).

    comm = FastComm(Topology(2, 4))            # one process per GPU (torchrun)
    recv = comm.alltoallv(send, send_counts)  # device bytes, stream-ordered
    all_to_all_fast(out, inp, out_splits, in_splits, comm=comm)

Per call, everything stays on the device (no host synchronisation):
  1. fast_gather_demand  P2P all-gather of the per-rank byte counts -> D
  2. fast_synth_batch    the FAST schedule for D (identical on every rank)
  3. fast_plan_compile   Appendix-A byte placement -> phase-ordered copy ops
  4. fast_exec           one persistent P2P kernel per rank over NVSwitch
The GPUs are split into virtual servers (n x m = world, e.g. 2x4 or 4x2):
phase 1 (balance) and the one-to-one stages both run over NVLink.

``GroupComm`` runs the same kernels for all ranks on ONE device (a
cooperative launch), used by the single-GPU parity tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .model import Topology, ValidationError, validate_topology
from .simulate import Timeline
from .synth import SynthBuffers, _device, _stream_handle

OP_DTYPE = np.dtype([("src_off", "<i8"), ("dst_off", "<i8"), ("len", "<i8"),
                     ("wait_off", "<i8"), ("sig_slot", "<i4"), ("wait_slot", "<i4"),
                     ("exec_rank", "<i2"), ("dst_rank", "<i2"), ("src_buf", "u1"),
                     ("dst_buf", "u1"), ("phase", "u1"), ("stage", "u1")])
PH_BALANCE, PH_DIRECT, PH_FROM_STAGING, PH_REDIST = 0, 1, 2, 3
BUF_SEND, BUF_RECV, BUF_STAGING = 0, 1, 2
TIMELINE_STRIDE = 16 + 4 * 256  # FAST_TIMELINE_STRIDE (include/fastb200.h)
TL_START, TL_BARRIER, TL_RECV_DONE, TL_BALANCE, TL_INTRA, TL_STAGE0 = 0, 1, 4, 8, 10, 16
STAGE_INTRA = 255
DEFAULT_BLOCKS = 128  # one 512-thread CTA per SM; must stay <= SM count (co-residency)
DEFAULT_CHUNK = 1024 * 1024


class _CudaBytes:
    """Zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def bytes_view(ptr: int, nbytes: int, device) -> torch.Tensor:
    return torch.as_tensor(_CudaBytes(ptr, nbytes), device=device)


class PlanBuffers:
    """Device buffers of one compiled plan (fast_plan)."""

    def __init__(self, n: int, m: int, device):
        lib = _lib.load()
        G = n * m
        self.capacity = int(lib.fast_plan_op_capacity(n, m))
        self.ops = torch.empty(self.capacity * OP_DTYPE.itemsize, dtype=torch.uint8, device=device)
        self.n_ops = torch.zeros(1, dtype=torch.int32, device=device)
        self.staging_used = torch.zeros(G, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.ws = torch.empty(int(lib.fast_plan_workspace_bytes(n, m)) + 16, dtype=torch.uint8,
                              device=device)
        self.struct = _lib.FastPlan(self.ops.data_ptr(), self.n_ops.data_ptr(),
                                    self.staging_used.data_ptr(), self.status.data_ptr(),
                                    self.ws.data_ptr(), self.capacity)

    def host_ops(self) -> np.ndarray:
        k = int(self.n_ops.item())
        return self.ops[: k * OP_DTYPE.itemsize].cpu().numpy().view(OP_DTYPE)


def plan_compile_host(D: np.ndarray, n: int, m: int, order: np.ndarray, perm: np.ndarray,
                      sbytes: np.ndarray, recv_cap: int, staging_cap: int,
                      send_self: np.ndarray | None = None, chunk: int = DEFAULT_CHUNK):
    """Host build of the plan logic (validation / inspection only)."""
    lib = _lib.load()
    D = np.ascontiguousarray(D, dtype=np.int64)
    K = n * n - 2 * n + 2
    perm_k = np.zeros((K, n), np.uint8)
    perm_k[: perm.shape[0]] = perm
    sb_k = np.zeros((K, n), np.int64)
    sb_k[: sbytes.shape[0]] = sbytes
    order = np.ascontiguousarray(order, dtype=np.int32)
    cap = int(lib.fast_plan_op_capacity(n, m))
    ops = np.zeros(cap, OP_DTYPE)
    n_ops = np.zeros(1, np.int32)
    used = np.zeros(n * m, np.int64)
    ws = np.zeros(int(lib.fast_plan_workspace_bytes(n, m)) + 16, np.uint8)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    ss = None if send_self is None else np.ascontiguousarray(send_self, dtype=np.int64)
    st = lib.fast_plan_compile_host(p(D), None if ss is None else p(ss), n, m,
                                    int(order.shape[0]), p(order), p(perm_k),
                                    p(sb_k), int(recv_cap), int(staging_cap), int(chunk),
                                    p(ops), cap,
                                    p(n_ops), p(used), p(ws))
    return ops[: int(n_ops[0])].copy(), used, int(st)


_NO_START = (1 << 64) - 1


def phase_windows(stamps: np.ndarray, n_stages: int) -> dict:
    """Measured (start, end) windows in seconds since the exec kernel's start,
    from one rank's timeline stamps (FAST_TL_* in include/fastb200.h); None
    for a phase this rank executed no chunk of."""
    u = stamps.astype(np.uint64)
    t0 = int(u[TL_START])

    def win(i):
        a, b = int(u[i]), int(u[i + 1])
        if a == _NO_START or b == 0:
            return None
        return ((a - t0) * 1e-9, (b - t0) * 1e-9)

    return {"barrier": (int(u[TL_BARRIER]) - t0) * 1e-9,
            "recv_done": (int(u[TL_RECV_DONE]) - t0) * 1e-9,
            "balance": win(TL_BALANCE), "intra": win(TL_INTRA),
            "scale_out": [win(TL_STAGE0 + 4 * k) for k in range(n_stages)],
            "redistribution": [win(TL_STAGE0 + 4 * k + 2) for k in range(n_stages)]}


def _n_stages_of(ops: np.ndarray | None) -> int:
    if ops is None or not len(ops):
        return 0
    st = ops["stage"][ops["stage"] != STAGE_INTRA]
    return int(st.max()) + 1 if len(st) else 0


def _timeline_from(stamps: np.ndarray, ops: np.ndarray | None, rank: int) -> Timeline:
    """Measured Timeline of one rank (the reference's phase breakdown,
    simulate.py:38-55): each phase's duration is its window on this rank
    (first chunk start to last chunk end); total = exec start -> this rank
    has sent its last chunk and every byte addressed to it has landed."""
    w = phase_windows(stamps, _n_stages_of(ops))
    dur = lambda x: 0.0 if x is None else max(0.0, x[1] - x[0])  # noqa: E731
    ends = [x[1] for x in [w["balance"], w["intra"], *w["scale_out"], *w["redistribution"]]
            if x is not None]
    return Timeline(t_balance=dur(w["balance"]), t_intra_a2a=dur(w["intra"]),
                    scale_out=tuple(dur(x) for x in w["scale_out"]),
                    redistribution=tuple(dur(x) for x in w["redistribution"]),
                    total=max([0.0, w["recv_done"], *ends]))


class FastComm:
    """One rank of the FAST executor (torch.distributed process group)."""

    def __init__(self, topology: Topology, recv_bytes: int, staging_bytes: int | None = None,
                 group=None, blocks: int = DEFAULT_BLOCKS, chunk_bytes: int = DEFAULT_CHUNK):
        import torch.distributed as dist

        validate_topology(topology)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if topology.gpu_count != self.world:
            raise ValidationError(f"topology {topology.n_servers}x{topology.gpus_per_server} "
                                  f"needs {topology.gpu_count} ranks, group has {self.world}")
        self.topology = topology
        self.device = _device()
        self.recv_bytes = int(recv_bytes)
        self.staging_bytes = int(staging_bytes if staging_bytes is not None else recv_bytes)
        self.blocks, self.chunk = blocks, chunk_bytes
        lib = _lib.load()
        ptr = ctypes.c_void_p()
        _lib.check_rc(lib.fast_comm_create(self.rank, self.world, 0, self.recv_bytes,
                                           self.staging_bytes, ctypes.byref(ptr)),
                      "fast_comm_create")
        self._ptr = ptr
        h = (ctypes.c_uint8 * 64)()
        _lib.check_rc(lib.fast_comm_ipc_handle(ptr, ctypes.cast(h, ctypes.c_void_p)),
                      "fast_comm_ipc_handle")
        handles: list = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=group)
        blob = b"".join(handles)
        _lib.check_rc(lib.fast_comm_open_peers(ptr, blob), "fast_comm_open_peers")
        dist.barrier(group=group)
        n, m = topology.n_servers, topology.gpus_per_server
        self.sched = SynthBuffers(1, n, m, self.device)
        self.plan = PlanBuffers(n, m, self.device)
        self.timeline = torch.zeros(TIMELINE_STRIDE, dtype=torch.int64, device=self.device)
        self.epoch = 0
        self.recv = bytes_view(lib.fast_comm_recv_ptr(ptr), self.recv_bytes, self.device)
        self._sched_ref = ctypes.byref(self.sched.struct)
        self._plan_ref = ctypes.byref(self.plan.struct)
        self.use_graph = True
        self._fused = False
        self._graphs: dict = {}
        self._count_cache: dict = {}
        self._split_bad: torch.Tensor | None = None
        self._copy_self = False  # state currently set in the C communicator

    def set_fused(self, enable: bool) -> None:
        """Single-launch path (gather + synthesis + plan inside the exec
        kernel, n <= 6) on/off; off by default (not faster on B200)."""
        _lib.check_rc(_lib.load().fast_comm_set_fused(self._ptr, 1 if enable else 0), "set_fused")
        self._fused = bool(enable)

    def set_pdl(self, enable: bool) -> None:
        """Programmatic dependent launch on the per-call kernel chain (on by
        default); cached call graphs are re-captured."""
        _lib.check_rc(_lib.load().fast_comm_set_pdl(self._ptr, 1 if enable else 0), "set_pdl")
        self._graphs.clear()

    def close(self) -> None:
        if getattr(self, "_ptr", None):
            _lib.load().fast_comm_destroy(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def demand(self) -> torch.Tensor:
        """The gathered G x G demand matrix of the last call (device)."""
        lib = _lib.load()
        ptr = lib.fast_comm_demand_ptr(self._ptr, 0)  # fixed slot: latest gathered matrix
        G = self.world
        return bytes_view(ptr, G * G * 8, self.device).view(torch.int64).view(G, G)

    def self_sizes(self) -> torch.Tensor:
        lib = _lib.load()
        ptr = lib.fast_comm_demand_ptr(self._ptr, 0) + 8 * self.world * self.world
        return bytes_view(ptr, self.world * 8, self.device).view(torch.int64)

    def _set_copy_self(self, enable: bool) -> None:
        if bool(enable) != self._copy_self:
            _lib.check_rc(_lib.load().fast_comm_set_copy_self(self._ptr, 1 if enable else 0),
                          "set_copy_self")
            self._copy_self = bool(enable)

    def alltoallv(self, send: torch.Tensor, send_counts: torch.Tensor,
                  stream: torch.cuda.Stream | None = None, record_timeline: bool = False,
                  exec_events: tuple | None = None,
                  send_rows: tuple | None = None, copy_self: bool = False) -> torch.Tensor:
        """FAST alltoallv of `send` (uint8, device) split by send_counts
        (int64[world] device, bytes per destination in send order; the own
        entry is the self segment, which stays in place and is not moved).
        Returns the recv region: source-major segments exactly like
        all_to_all_single's output, except that the own segment's slot is a
        gap of send_counts[rank] bytes (never transferred; fill it locally).

        send_rows = (rows, row_src, row_bytes): the send buffer is virtual,
        its row r being row row_src[r] of `rows` (fused MoE pack -> send,
        fast_comm_set_send_rows); `send` is then only a placeholder."""
        lib = _lib.load()
        self._set_copy_self(copy_self)
        if send_rows is None:
            return self._alltoallv(send, send_counts, stream, record_timeline, exec_events)
        rows, row_src, row_bytes = send_rows
        if row_src.dtype != torch.int32 or not row_src.is_cuda or not rows.is_cuda:
            raise ValidationError("send_rows: rows / row_src (int32) must be cuda tensors")
        _lib.check_rc(lib.fast_comm_set_send_rows(self._ptr, ctypes.c_void_p(rows.data_ptr()),
                                                  ctypes.c_void_p(row_src.data_ptr()),
                                                  int(row_bytes), row_src.numel()),
                      "fast_comm_set_send_rows")
        try:
            return self._alltoallv(send, send_counts, stream, record_timeline, exec_events,
                                   (rows.data_ptr(), row_src.data_ptr(), int(row_bytes)),
                                   send_cap=int(row_src.numel()) * int(row_bytes))
        finally:
            lib.fast_comm_set_send_rows(self._ptr, None, None, 0, 0)

    def _alltoallv(self, send, send_counts, stream, record_timeline, exec_events,
                   rows_key=None, send_cap=None) -> torch.Tensor:
        lib = _lib.load()
        if send.dtype != torch.uint8 or not send.is_cuda:
            raise ValidationError("send must be a cuda uint8 tensor")
        n, m = self.topology.n_servers, self.topology.gpus_per_server
        s = stream or torch.cuda.current_stream()
        row = send_counts
        if row.dtype != torch.int64 or row.device != self.device or not row.is_contiguous():
            with torch.cuda.stream(s):  # converted on the stream that consumes it
                row = row.to(device=self.device, dtype=torch.int64).contiguous()
        self._row = row  # keep alive until the stream consumes it
        cap = int(send.numel()) if send_cap is None else int(send_cap)
        _lib.check_rc(lib.fast_comm_set_send_capacity(self._ptr, cap), "set_send_capacity")
        tl = ctypes.c_void_p(self.timeline.data_ptr()) if record_timeline else None
        if exec_events is None:
            key = (send.data_ptr(), cap, row.data_ptr(), bool(record_timeline), self._fused,
                   rows_key, self._copy_self)
            g = self._graphs.get(key) if (self.use_graph and stream is None) else None
            if g is not None:  # one graph launch per call
                g.replay()
                self.epoch += 1
                return self.recv
            lib.fast_comm_set_epoch(self._ptr, self.epoch)  # graph replays bypass the host mirror
            _lib.check_rc(lib.fast_alltoallv(self._ptr, ctypes.c_void_p(send.data_ptr()),
                                             ctypes.c_void_p(row.data_ptr()), n, m,
                                             self._sched_ref, self._plan_ref, self.blocks,
                                             self.chunk, tl, ctypes.c_void_p(s.cuda_stream)),
                          "fast_alltoallv")
            self.epoch += 1
            if self.use_graph and stream is None and len(self._graphs) < 16:
                self._capture(key, send, row, tl)
            return self.recv
        # step by step (exec-kernel events for the benchmark)
        self.epoch += 1
        sh = ctypes.c_void_p(s.cuda_stream)
        _lib.check_rc(lib.fast_gather_demand(self._ptr, ctypes.c_void_p(row.data_ptr()),
                                             self.epoch, sh), "fast_gather_demand")
        dptr = lib.fast_comm_demand_ptr(self._ptr, self.epoch)
        _lib.check_rc(lib.fast_synth_batch(ctypes.c_void_p(dptr), 1, n, m,
                                           ctypes.byref(self.sched.struct), sh), "fast_synth_batch")
        sself = ctypes.c_void_p(dptr + 8 * self.world * self.world)
        _lib.check_rc(lib.fast_plan_compile_ex(ctypes.c_void_p(dptr), sself, n, m,
                                               ctypes.byref(self.sched.struct), self.recv_bytes,
                                               self.staging_bytes, self.chunk,
                                               ctypes.byref(self.plan.struct),
                                               1 if self._copy_self else 0, sh),
                      "fast_plan_compile_ex")
        exec_events[0].record(s)
        _lib.check_rc(lib.fast_exec(self._ptr, ctypes.byref(self.plan.struct),
                                    ctypes.c_void_p(send.data_ptr()), self.epoch, self.blocks,
                                    self.chunk, tl, sh), "fast_exec")
        exec_events[1].record(s)
        _lib.check_rc(lib.fast_comm_set_epoch(self._ptr, self.epoch), "fast_comm_set_epoch")
        return self.recv

    def _capture(self, key, send: torch.Tensor, row: torch.Tensor, tl) -> None:
        """Capture fast_alltoallv for this (send, counts) pair into a CUDA
        graph (capture only records; the call above did the work)."""
        lib = _lib.load()
        n, m = self.topology.n_servers, self.topology.gpus_per_server
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cs = torch.cuda.current_stream()
            rc = lib.fast_alltoallv(self._ptr, ctypes.c_void_p(send.data_ptr()),
                                    ctypes.c_void_p(row.data_ptr()), n, m, self._sched_ref,
                                    self._plan_ref, self.blocks, self.chunk, tl,
                                    ctypes.c_void_p(cs.cuda_stream))
        _lib.check_rc(rc, "fast_alltoallv (capture)")
        lib.fast_comm_set_epoch(self._ptr, self.epoch)  # capture did not execute
        self._graphs[key] = g

    def check(self) -> None:
        """Raise if the last call's device status reports a failure (syncs)."""
        st = ctypes.c_int32()
        _lib.check_rc(_lib.load().fast_comm_status(self._ptr, ctypes.byref(st)), "status")
        plan_st = int(self.plan.status.item())
        if plan_st != 0:
            _lib.check_rc(plan_st, "fast_plan_compile")
        if st.value == 2:
            raise ValidationError("fast_exec: send counts overrun the send buffer "
                                  "(recreate the communicator)")
        if st.value != 0:
            _lib.check_rc(3, "fast_exec (timeout / protocol; recreate the communicator)")
        if self._split_bad is not None and bool(self._split_bad.item()):
            raise ValidationError("all_to_all_fast: output_split_sizes disagree with the "
                                  "gathered send counts")

    def _counts_for(self, splits: tuple, row_bytes: int, out: bool = False) -> torch.Tensor:
        """Device int64 bytes-per-rank vector for a split tuple, cached (no
        per-call host->device copy; stable pointers keep the call graphs)."""
        key = (splits, int(row_bytes), out)
        t = self._count_cache.get(key)
        if t is None:
            h = torch.tensor([int(x) * int(row_bytes) for x in splits], dtype=torch.int64)
            t = h.pin_memory().to(self.device, non_blocking=True)
            if len(self._count_cache) > 256:
                self._count_cache.clear()
            self._count_cache[key] = t
        return t

    def _check_output_splits(self, out_bytes: torch.Tensor) -> None:
        """Device-side: the gathered column `rank` (bytes each source sends
        here, own segment from the self sizes) must equal out_bytes; a
        mismatch is recorded and raised by check()."""
        r = self.rank
        col = self.demand()[:, r].clone()
        col[r] = self.self_sizes()[r]
        bad = (col != out_bytes).any()
        if self._split_bad is None:
            self._split_bad = bad.clone()
        else:
            self._split_bad.logical_or_(bad)

    def measured_timeline(self) -> Timeline:
        """Timeline of the last call made with record_timeline=True (syncs)."""
        return _timeline_from(self.timeline.cpu().numpy(), self.plan.host_ops(), self.rank)

    def measured_phases(self) -> dict:
        """(start, end) phase windows of the last recorded call (syncs)."""
        return phase_windows(self.timeline.cpu().numpy(), _n_stages_of(self.plan.host_ops()))


def all_to_all_fast(output: torch.Tensor | None, input: torch.Tensor,
                    output_split_sizes: list[int] | None = None,
                    input_split_sizes: list[int] | None = None,
                    comm: FastComm | None = None, check_splits: bool = True) -> torch.Tensor:
    """Drop-in for torch.distributed.all_to_all_single on the
    FAST path.  Splits are along dim 0 in rows.

    The executor writes every remote segment straight into the
    communicator's receive region, laid out exactly like all_to_all_single's
    output with a gap at the own slot; the own segment is one local copy into
    that gap.  ``output=None`` returns that region as the result (zero copy;
    valid until the next call on `comm`); a caller-owned `output` receives one
    contiguous device copy.  Split counts are cached on the device (no
    per-call host->device copy).  check_splits: output_split_sizes are
    compared on the device with the gathered send counts; a mismatch is
    raised by comm.check()."""
    if comm is None:
        raise ValidationError("all_to_all_fast needs a FastComm")
    W = comm.world
    rows_in = input.shape[0]
    row_bytes = (input[0].numel() if rows_in else
                 int(np.prod(input.shape[1:], dtype=np.int64))) * input.element_size()
    if input_split_sizes is None:
        if rows_in % W:
            raise ValidationError("input rows are not divisible by the world size")
        input_split_sizes = [rows_in // W] * W
    if output_split_sizes is None:
        if output is None:
            raise ValidationError("output_split_sizes are needed without an output tensor")
        if output.shape[0] % W:
            raise ValidationError("output rows are not divisible by the world size")
        output_split_sizes = [output.shape[0] // W] * W
    if len(input_split_sizes) != W or len(output_split_sizes) != W:
        raise ValidationError("split lists must have one entry per rank")
    if sum(input_split_sizes) != rows_in:
        raise ValidationError("input_split_sizes do not sum to the input rows")
    total_out = sum(output_split_sizes) * row_bytes
    if total_out > comm.recv_bytes:
        raise ValidationError("output larger than the communicator's receive region")
    if output is not None and output.numel() * output.element_size() < total_out:
        raise ValidationError("output tensor smaller than sum(output_split_sizes)")
    inb = input.contiguous().view(torch.uint8).reshape(-1)
    counts = comm._counts_for(tuple(input_split_sizes), row_bytes)
    # the exec CTAs also move the own segment into its slot (a local op next
    # to the remote sends), so the region is the complete output
    recv = comm.alltoallv(inb, counts, copy_self=True)
    if check_splits:
        comm._check_output_splits(comm._counts_for(tuple(output_split_sizes), row_bytes, True))
    res = recv[:total_out].view(input.dtype).view(-1, *input.shape[1:])
    if output is None:
        return res
    if total_out:
        output.view(torch.uint8).reshape(-1)[:total_out].copy_(recv[:total_out])
    return output


class _AllToAllFast(torch.autograd.Function):
    """all_to_all_fast with autograd: the backward is the reverse FAST
    alltoallv of the output gradient (the transposed demand matrix D^T: the
    split lists swap roles), as for all_to_all_single."""

    @staticmethod
    def forward(ctx, input, output_split_sizes, input_split_sizes, comm, bwd_comm):
        ctx.splits = (list(output_split_sizes), list(input_split_sizes))
        ctx.comm = bwd_comm or comm
        out = torch.empty((sum(output_split_sizes),) + tuple(input.shape[1:]), dtype=input.dtype,
                          device=input.device)
        return all_to_all_fast(out, input, output_split_sizes, input_split_sizes, comm=comm)

    @staticmethod
    def backward(ctx, grad):
        out_s, in_s = ctx.splits
        g = grad.contiguous()
        gin = torch.empty((sum(in_s),) + tuple(g.shape[1:]), dtype=g.dtype, device=g.device)
        all_to_all_fast(gin, g, in_s, out_s, comm=ctx.comm)
        return gin, None, None, None, None


def all_to_all_fast_autograd(input: torch.Tensor, output_split_sizes: list[int],
                             input_split_sizes: list[int], comm: FastComm,
                             bwd_comm: FastComm | None = None) -> torch.Tensor:
    """Differentiable all_to_all_fast (returns a new tensor; the backward runs
    on `bwd_comm`, default `comm`)."""
    return _AllToAllFast.apply(input, output_split_sizes, input_split_sizes, comm, bwd_comm)


class GroupRank:
    """Rank view of a GroupComm (world, rank, device) for per-rank helpers
    such as MoEDispatch in single-GPU tests."""

    def __init__(self, group: "GroupComm", rank: int):
        self.world, self.rank, self.device = group.world, rank, group.device
        self.recv = group.recvs[rank]


class GroupComm:
    """All `world` ranks on ONE device: same plan + exec kernels, launched as
    one cooperative kernel (tests, single-GPU benchmarks of the protocol)."""

    def __init__(self, topology: Topology, recv_bytes: int, staging_bytes: int | None = None,
                 blocks: int = 8, chunk_bytes: int = DEFAULT_CHUNK):
        validate_topology(topology)
        self.topology = topology
        self.world = topology.gpu_count
        self.device = _device()
        self.recv_bytes = int(recv_bytes)
        self.staging_bytes = int(staging_bytes if staging_bytes is not None else recv_bytes)
        self.blocks, self.chunk = blocks, chunk_bytes
        lib = _lib.load()
        arr = (ctypes.c_void_p * self.world)()
        _lib.check_rc(lib.fast_comm_create_group(self.world, self.recv_bytes, self.staging_bytes,
                                                 arr), "fast_comm_create_group")
        self._ptrs = arr
        n, m = topology.n_servers, topology.gpu_count // topology.n_servers
        self.sched = SynthBuffers(1, n, m, self.device)
        self.plan = PlanBuffers(n, m, self.device)
        self.timeline = torch.zeros(self.world * TIMELINE_STRIDE, dtype=torch.int64,
                                    device=self.device)
        self.epoch = 0
        self.recvs = [bytes_view(lib.fast_comm_recv_ptr(ctypes.c_void_p(p)), self.recv_bytes,
                                 self.device) for p in arr]

    def close(self) -> None:
        if getattr(self, "_ptrs", None) is not None:
            lib = _lib.load()
            for p in self._ptrs:
                lib.fast_comm_destroy(ctypes.c_void_p(p))
            self._ptrs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alltoallv(self, sends: list[torch.Tensor], D: torch.Tensor,
                  stream: torch.cuda.Stream | None = None,
                  self_bytes: torch.Tensor | None = None,
                  send_rows: list | None = None,
                  exec_events: tuple | None = None,
                  copy_self: bool = False) -> list[torch.Tensor]:
        """D: [world, world] int64, zero diagonal.  self_bytes (optional,
        int64[world]): own segments kept in place in send_g and left as a
        gap in recv_g (all_to_all_single layout).  send_rows (optional, per
        rank (rows, row_src, row_bytes)): row-mapped send buffers, as in
        FastComm.alltoallv."""
        lib = _lib.load()
        if send_rows is not None:
            for r, (rows, row_src, rb) in enumerate(send_rows):
                _lib.check_rc(lib.fast_comm_set_send_rows(
                    self._ptrs[r], ctypes.c_void_p(rows.data_ptr()),
                    ctypes.c_void_p(row_src.data_ptr()), int(rb), row_src.numel()),
                    "fast_comm_set_send_rows")
            try:
                return self.alltoallv(sends, D, stream, self_bytes, exec_events=exec_events,
                                      copy_self=copy_self)
            finally:
                for r in range(self.world):
                    lib.fast_comm_set_send_rows(self._ptrs[r], None, None, 0, 0)
        n, m = self.topology.n_servers, self.topology.gpus_per_server
        if D.dtype != torch.int64 or tuple(D.shape) != (self.world, self.world):
            raise ValidationError("D must be int64 [world, world]")
        self._D = D.to(self.device).contiguous()
        self._self = None if self_bytes is None else self_bytes.to(self.device, torch.int64).contiguous()
        self.epoch += 1
        sh = _stream_handle(stream)
        dp = ctypes.c_void_p(self._D.data_ptr())
        _lib.check_rc(lib.fast_synth_batch(dp, 1, n, m, ctypes.byref(self.sched.struct), sh),
                      "fast_synth_batch")
        sp_self = None if self._self is None else ctypes.c_void_p(self._self.data_ptr())
        _lib.check_rc(lib.fast_plan_compile_ex(dp, sp_self, n, m, ctypes.byref(self.sched.struct),
                                               self.recv_bytes, self.staging_bytes, self.chunk,
                                               ctypes.byref(self.plan.struct),
                                               1 if copy_self else 0, sh),
                      "fast_plan_compile_ex")
        sp = (ctypes.c_void_p * self.world)(*[s.data_ptr() for s in sends])
        if exec_events is not None:
            exec_events[0].record(stream or torch.cuda.current_stream())
        _lib.check_rc(lib.fast_exec_group(self._ptrs, self.world, ctypes.byref(self.plan.struct),
                                          sp, self.epoch, self.blocks, self.chunk,
                                          ctypes.c_void_p(self.timeline.data_ptr()), sh),
                      "fast_exec_group")
        if exec_events is not None:
            exec_events[1].record(stream or torch.cuda.current_stream())
        return self.recvs

    def measured_timeline(self, rank: int) -> Timeline:
        """Measured Timeline of `rank` in the last call (syncs)."""
        st = self.timeline.view(self.world, TIMELINE_STRIDE)[rank].cpu().numpy()
        return _timeline_from(st, self.plan.host_ops(), rank)

    def measured_phases(self, rank: int) -> dict:
        st = self.timeline.view(self.world, TIMELINE_STRIDE)[rank].cpu().numpy()
        return phase_windows(st, _n_stages_of(self.plan.host_ops()))

    def check(self) -> None:
        lib = _lib.load()
        plan_st = int(self.plan.status.item())
        if plan_st != 0:
            _lib.check_rc(plan_st, "fast_plan_compile")
        for p in self._ptrs:
            st = ctypes.c_int32()
            _lib.check_rc(lib.fast_comm_status(ctypes.c_void_p(p), ctypes.byref(st)), "status")
            if st.value != 0:
                _lib.check_rc(3, "fast_exec_group (timeout / protocol)")


def execute_fast(comm: FastComm, send: torch.Tensor, send_counts: torch.Tensor) -> torch.Tensor:
    """Alias of comm.alltoallv (the executor behind simulate_fast's API)."""
    return comm.alltoallv(send, send_counts)
