"""MoE dispatch front-end: gating -> histogram/scan -> pack -> FAST
alltoallv -> unpack, all on the device (BASELINE config 3).

    disp = MoEDispatch(comm, tokens_per_gpu=16384, row_bytes=8192)
    expert_in = disp.dispatch(tokens, seed=0)   # [recv rows, row_bytes] uint8

Rank r hosts experts [r*L, (r+1)*L) (E = L * world).  The receive region of the executor is
laid out like all_to_all_single's output with a gap at the self slot; the
unpack kernel copies the local segment into that gap, so the receive region
IS the expert input (source-major, stable token order within a source).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .model import ValidationError
from .synth import _stream_handle


def gating_thresholds(E: int, alpha: float = 0.8, hot: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Integer CDF thresholds of w_e = 1/((e-hot) mod E + 1)^alpha (top-1) and,
    per first choice e, of w with w[e] = 0 (top-2)."""
    w = 1.0 / (((np.arange(E) - hot) % E) + 1.0) ** alpha

    def cdf(x):
        t = np.floor(np.cumsum(x) / x.sum() * 2.0 ** 32).astype(np.uint64)
        t[-1] = np.uint64(1 << 32)
        return t

    return cdf(w), np.stack([cdf(np.where(np.arange(E) == e, 0.0, w)) for e in range(E)])


class MoEDispatch:
    """Device buffers + the kernels of one MoE dispatch (one rank).

    num_experts E (default: the world size) must be a multiple of the world
    W; rank r hosts experts [r*L, (r+1)*L), L = E / W.  The top-k expert ids
    come from the caller's router (``dispatch(tokens, topk=...)``, int32
    [T, k], k in 1/2/4/8) or, for benchmarks, from the deterministic
    synthetic top-2 gate (``dispatch(tokens, seed=...)``).  The send layout
    is expert-major (Megatron's permute order), so each destination rank
    receives, per source, its experts' rows expert by expert."""

    def __init__(self, comm, tokens_per_gpu: int, row_bytes: int, k: int = 2,
                 alpha: float = 0.8, fused_pack: bool = False, num_experts: int | None = None,
                 exec_self: bool = True):
        if row_bytes % 16:
            raise ValidationError("row_bytes must be a multiple of 16")
        if k not in (1, 2, 4, 8):
            raise ValidationError("top-k must be 1, 2, 4 or 8")
        self.comm = comm
        self.T, self.row_bytes, self.k = tokens_per_gpu, row_bytes, k
        self.E = int(num_experts or comm.world)
        if self.E % comm.world or self.E > 64:
            raise ValidationError(f"num_experts {self.E} must be a multiple of the world size "
                                  f"{comm.world} and <= 64")
        self.L = self.E // comm.world
        dev = comm.device
        lib = _lib.load()
        self._gate_topk = torch.empty(self.T * k, dtype=torch.int32, device=dev)
        self.topk = self._gate_topk  # the ids of the last route (gate's or the router's)
        self.pos = torch.empty(self.T * k, dtype=torch.int32, device=dev)
        self.counts = torch.empty(self.E, dtype=torch.int64, device=dev)
        self.seg_rows = torch.empty(self.E, dtype=torch.int64, device=dev)
        self.demand_row = torch.empty(comm.world, dtype=torch.int64, device=dev)
        self.ws = torch.empty(max(16, int(lib.fast_moe_route_workspace_bytes(self.T, k, self.E))),
                              dtype=torch.uint8, device=dev)
        # fused_pack: the executor reads token rows through row_src (4 B per
        # send row) and the packed send buffer is never written
        self.fused_pack = fused_pack
        self.row_src = torch.empty(self.T * k, dtype=torch.int32, device=dev)
        self.send = torch.empty(0 if fused_pack else self.T * k * row_bytes, dtype=torch.uint8,
                                device=dev)
        # FastComm: the exec kernel copies the own segment (FAST_PLAN_COPY_SELF);
        # group-mode rank views keep the explicit unpack
        self.exec_self = exec_self and hasattr(comm, "_set_copy_self")
        self.set_hot(0, alpha)

    def set_hot(self, hot: int, alpha: float = 0.8) -> None:
        thr, thr2 = gating_thresholds(self.E, alpha, hot)
        self.thr = torch.from_numpy(thr.view(np.int64)).to(self.comm.device)
        self.thr2 = torch.from_numpy(np.ascontiguousarray(thr2).view(np.int64)).to(self.comm.device)

    def route(self, seed: int | None = None, stream=None,
              topk: torch.Tensor | None = None) -> None:
        """Top-k ids (the router's, or the synthetic gate's for `seed`) ->
        histogram / scan: stable send rows, per-expert counts and this rank's
        row of the demand matrix (the traffic-matrix builder)."""
        lib = _lib.load()
        sh = _stream_handle(stream)
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        if topk is not None:
            if (topk.dtype != torch.int32 or not topk.is_cuda
                    or topk.numel() != self.T * self.k):
                raise ValidationError(f"topk must be a cuda int32 tensor [{self.T}, {self.k}]")
            self.topk = topk.contiguous().view(-1)
        else:
            if seed is None:
                raise ValidationError("route needs the router's topk or a gate seed")
            if self.k != 2:
                raise ValidationError("the synthetic gate is top-2; pass the router's topk")
            self.topk = self._gate_topk  # never write into a router's tensor
            _lib.check_rc(lib.fast_moe_gate(self.T, ctypes.c_uint64(seed * 1000 + self.comm.rank),
                                            self.E, P(self.thr), P(self.thr2), P(self.topk), sh),
                          "fast_moe_gate")
        _lib.check_rc(lib.fast_moe_route_ex(P(self.topk), self.T, self.k, self.E, self.L,
                                            self.row_bytes, P(self.pos), P(self.counts),
                                            P(self.seg_rows), P(self.demand_row), P(self.ws), sh),
                      "fast_moe_route_ex")

    def pack(self, tokens: torch.Tensor, stream=None) -> None:
        lib = _lib.load()
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        if tokens.numel() * tokens.element_size() != self.T * self.row_bytes:
            raise ValidationError("tokens must be [T, row_bytes] worth of data")
        _lib.check_rc(lib.fast_moe_pack(P(tokens), self.T, self.k, self.row_bytes, P(self.topk),
                                        P(self.pos), P(self.ws), self.E, P(self.seg_rows),
                                        P(self.send), _stream_handle(stream)), "fast_moe_pack")

    def rowmap(self, stream=None, tokens: torch.Tensor | None = None) -> None:
        """row_src[send row] = token (fast_moe_rowmap): the pack's
        destination map inverted, for the fused pack -> send.  `tokens`
        (kept for unpack) defaults to the last dispatch's."""
        lib = _lib.load()
        if tokens is not None:
            if tokens.numel() * tokens.element_size() != self.T * self.row_bytes:
                raise ValidationError("tokens must be [T, row_bytes] worth of data")
            self._tokens = tokens.contiguous().view(torch.uint8).reshape(-1)
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check_rc(lib.fast_moe_rowmap(self.T, self.k, P(self.topk), P(self.pos), P(self.ws),
                                          self.E, P(self.seg_rows), P(self.row_src),
                                          _stream_handle(stream)), "fast_moe_rowmap")

    def unpack(self, stream=None, D: torch.Tensor | None = None,
               self_sizes: torch.Tensor | None = None, recv: torch.Tensor | None = None
               ) -> torch.Tensor:
        """Copy the own segment into the self slot of the receive region.
        D / self_sizes / recv default to the communicator's last call."""
        lib = _lib.load()
        c = self.comm
        D = c.demand() if D is None else D
        ss = c.self_sizes() if self_sizes is None else self_sizes
        recv = c.recv if recv is None else recv
        if self.fused_pack:
            P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
            _lib.check_rc(lib.fast_moe_unpack_self_rows(P(D), P(ss), c.world, c.rank,
                                                        P(self._tokens), P(self.row_src),
                                                        self.row_bytes, P(recv),
                                                        _stream_handle(stream)),
                          "fast_moe_unpack_self_rows")
            return recv
        _lib.check_rc(lib.fast_moe_unpack_self(ctypes.c_void_p(D.data_ptr()),
                                               ctypes.c_void_p(ss.data_ptr()), c.world, c.rank,
                                               ctypes.c_void_p(self.send.data_ptr()),
                                               ctypes.c_void_p(recv.data_ptr()),
                                               _stream_handle(stream)), "fast_moe_unpack_self")
        return recv

    def dispatch(self, tokens: torch.Tensor, seed: int | None = None, stream=None,
                 topk: torch.Tensor | None = None) -> torch.Tensor:
        """Full dispatch; returns the receive region (expert input rows,
        source-major; per source this rank's experts in order; the row count
        is this rank's experts' counts summed over sources)."""
        self.route(seed, stream, topk)
        # the own experts' rows: moved by the exec CTAs next to the remote
        # sends (a local op of the plan) instead of a separate unpack after it
        kw = {"copy_self": True} if self.exec_self else {}
        if self.fused_pack:
            self.rowmap(stream, tokens)
            self.comm.alltoallv(self._tokens, self.demand_row, stream=stream,
                                send_rows=(self._tokens, self.row_src, self.row_bytes), **kw)
        else:
            self.pack(tokens, stream)
            self.comm.alltoallv(self.send, self.demand_row, stream=stream, **kw)
        # the demand matrix lands on `stream`: snapshot it there (not on the
        # current stream, which may run ahead of a side stream)
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.remember_forward(self.comm.demand(), self.comm.self_sizes())
        if self.exec_self:
            return self.comm.recv
        return self.unpack(stream)

    def remember_forward(self, D: torch.Tensor, self_sizes: torch.Tensor) -> None:
        """Keep the forward call's demand matrix: the combine sends column
        `rank` of it back (D^T), self segment kept local."""
        r = self.comm.rank
        self.Dfwd = D.clone()
        self.comb_counts = D[:, r].clone()
        self.comb_counts[r] = self_sizes[r]

    def tokens_per_expert(self) -> torch.Tensor:
        """[world, L] rows this rank received per (source, local expert) in
        the last dispatch (Megatron's num_global_tokens_per_expert slice).
        Uses the process group (FastComm only)."""
        import torch.distributed as dist

        allc = torch.empty(self.comm.world, self.E, dtype=torch.int64, device=self.comm.device)
        dist.all_gather_into_tensor(allc, self.counts)
        r, L = self.comm.rank, self.L
        return allc[:, r * L:(r + 1) * L]

    def combine_rows(self, comb_recv: torch.Tensor, expert_out: torch.Tensor,
                     weights: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
        """Weighted un-permute of the combine receive buffer into token order
        (fast_moe_combine); `out` is [T, row_bytes/2] bf16."""
        lib = _lib.load()
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        if weights.dtype != torch.float32 or weights.numel() != self.T * self.k:
            raise ValidationError("weights must be float32 [T, k]")
        if out.dtype != torch.bfloat16 or out.numel() * 2 != self.T * self.row_bytes:
            raise ValidationError("out must be bf16 [T, row_bytes/2]")
        _lib.check_rc(lib.fast_moe_combine_ex(P(comb_recv), P(expert_out), P(self.Dfwd),
                                              self.comm.world, self.comm.rank, self.T, self.k,
                                              self.row_bytes, P(self.topk), P(self.pos),
                                              P(self.ws), self.E, self.L, P(self.seg_rows),
                                              P(weights.contiguous()), P(out),
                                              _stream_handle(stream)), "fast_moe_combine_ex")
        return out

    def combine(self, expert_out: torch.Tensor, weights: torch.Tensor, out: torch.Tensor,
                stream=None) -> torch.Tensor:
        """Reverse FAST alltoallv of the expert outputs (forward receive
        layout; must not alias the communicator's receive region) and the
        weighted top-k combine back into token order."""
        if expert_out.data_ptr() == self.comm.recv.data_ptr():
            raise ValidationError("expert_out must not alias the receive region")
        recv = self.comm.alltoallv(expert_out.view(torch.uint8).reshape(-1), self.comb_counts,
                                   stream=stream)
        return self.combine_rows(recv, expert_out, weights, out, stream)
