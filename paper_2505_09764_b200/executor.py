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
TIMELINE_STRIDE = 8 + 256
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


def _timeline_from(stamps: np.ndarray, ops: np.ndarray | None, rank: int) -> Timeline:
    t0 = stamps[1]
    sec = lambda x: max(0.0, (int(x) - int(t0)) * 1e-9) if x else 0.0  # noqa: E731
    n_st = 0
    if ops is not None and len(ops):
        n_st = int(ops["stage"].max()) + 1
    so = tuple(sec(stamps[8 + k]) for k in range(n_st))
    return Timeline(t_balance=sec(stamps[2]), t_intra_a2a=0.0, scale_out=so,
                    redistribution=tuple(0.0 for _ in so), total=sec(stamps[4]))


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

    def set_fused(self, enable: bool) -> None:
        """Single-launch path (gather + synthesis + plan inside the exec
        kernel, n <= 6) on/off; off by default (not faster on B200)."""
        _lib.check_rc(_lib.load().fast_comm_set_fused(self._ptr, 1 if enable else 0), "set_fused")
        self._fused = bool(enable)

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

    def alltoallv(self, send: torch.Tensor, send_counts: torch.Tensor,
                  stream: torch.cuda.Stream | None = None, record_timeline: bool = False,
                  exec_events: tuple | None = None,
                  send_rows: tuple | None = None) -> torch.Tensor:
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
                                   (rows.data_ptr(), row_src.data_ptr(), int(row_bytes)))
        finally:
            lib.fast_comm_set_send_rows(self._ptr, None, None, 0, 0)

    def _alltoallv(self, send, send_counts, stream, record_timeline, exec_events,
                   rows_key=None) -> torch.Tensor:
        lib = _lib.load()
        if send.dtype != torch.uint8 or not send.is_cuda:
            raise ValidationError("send must be a cuda uint8 tensor")
        n, m = self.topology.n_servers, self.topology.gpus_per_server
        row = send_counts
        if row.dtype != torch.int64 or row.device != self.device or not row.is_contiguous():
            row = row.to(device=self.device, dtype=torch.int64).contiguous()
        self._row = row  # keep alive until the stream consumes it
        s = stream or torch.cuda.current_stream()
        tl = ctypes.c_void_p(self.timeline.data_ptr()) if record_timeline else None
        if exec_events is None:
            key = (send.data_ptr(), row.data_ptr(), bool(record_timeline), self._fused, rows_key)
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
        _lib.check_rc(lib.fast_plan_compile(ctypes.c_void_p(dptr), sself, n, m,
                                            ctypes.byref(self.sched.struct), self.recv_bytes,
                                            self.staging_bytes, self.chunk,
                                            ctypes.byref(self.plan.struct), sh),
                      "fast_plan_compile")
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
        if st.value != 0:
            _lib.check_rc(3, "fast_exec (timeout / protocol)")

    def measured_timeline(self) -> Timeline:
        return _timeline_from(self.timeline.cpu().numpy(), self.plan.host_ops(), self.rank)


def all_to_all_fast(output: torch.Tensor, input: torch.Tensor,
                    output_split_sizes: list[int] | None = None,
                    input_split_sizes: list[int] | None = None,
                    comm: FastComm | None = None) -> torch.Tensor:
    """Drop-in for torch.distributed.all_to_all_single on the
    FAST path.  Splits are along dim 0 in rows; the self segment is a local
    copy, everything else goes through comm.alltoallv."""
    if comm is None:
        raise ValidationError("all_to_all_fast needs a FastComm")
    W = comm.world
    rows_in, rows_out = input.shape[0], output.shape[0]
    row_bytes = input[0].numel() * input.element_size() if rows_in else 0
    if input_split_sizes is None:
        input_split_sizes = [rows_in // W] * W
    if output_split_sizes is None:
        output_split_sizes = [rows_out // W] * W
    inb = input.contiguous().view(torch.uint8).reshape(-1)
    counts = torch.tensor([s * row_bytes for s in input_split_sizes], dtype=torch.int64,
                          device=input.device)
    recv = comm.alltoallv(inb, counts)
    # recv is laid out like all_to_all_single's output with a gap at the self
    # slot: one contiguous copy, then the local segment into its slot
    outb = output.view(torch.uint8).reshape(-1)
    r = comm.rank
    total_out = sum(output_split_sizes) * row_bytes
    self_in = sum(input_split_sizes[:r]) * row_bytes
    self_out = sum(output_split_sizes[:r]) * row_bytes
    nself = input_split_sizes[r] * row_bytes
    if total_out:
        outb[:total_out].copy_(recv[:total_out])
    if nself:
        outb[self_out:self_out + nself].copy_(inb[self_in:self_in + nself])
    return output


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
                  send_rows: list | None = None) -> list[torch.Tensor]:
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
                return self.alltoallv(sends, D, stream, self_bytes)
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
        _lib.check_rc(lib.fast_plan_compile(dp, sp_self, n, m, ctypes.byref(self.sched.struct),
                                            self.recv_bytes, self.staging_bytes, self.chunk,
                                            ctypes.byref(self.plan.struct), sh),
                      "fast_plan_compile")
        sp = (ctypes.c_void_p * self.world)(*[s.data_ptr() for s in sends])
        _lib.check_rc(lib.fast_exec_group(self._ptrs, self.world, ctypes.byref(self.plan.struct),
                                          sp, self.epoch, self.blocks, self.chunk,
                                          ctypes.c_void_p(self.timeline.data_ptr()), sh),
                      "fast_exec_group")
        return self.recvs

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
