"""ctypes binding of libfastb200.so (the C-ABI in include/fastb200.h).

There is no fallback: if the library is missing or a symbol is absent the
import of the GPU entry points raises ``RuntimeError``.  Nothing here depends
on torch; callers pass raw device pointers (``tensor.data_ptr()``) and a
stream handle (``torch.cuda.current_stream().cuda_stream``).
"""

from __future__ import annotations

import ctypes
import os

from ._build import LIB_PATH

FAST_OK = 0
FAST_EVALIDATION = 2
FAST_EINVARIANT = 3
FAST_ECUDA = -1
FAST_MAX_SERVERS = 128
FAST_MAX_GPUS_PER_SERVER = 64
FAST_DEC_SERVER = 0
FAST_DEC_DOUBLY_STOCHASTIC = 1

c_i64p = ctypes.POINTER(ctypes.c_int64)


class FastMove(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_int64), ("from_gpu", ctypes.c_int32),
                ("to_gpu", ctypes.c_int32)]


class FastSchedBufs(ctypes.Structure):
    """Mirror of ``fast_sched_bufs`` (all device pointers)."""

    _fields_ = [(name, ctypes.c_void_p) for name in (
        "balanced", "server", "move_count", "moves", "common_sum", "aux",
        "n_raw", "stage_weight", "stage_perm", "stage_bytes", "n_stages",
        "stage_order", "status", "workspace", "strip", "tile_mask")]


class FastPlan(ctypes.Structure):
    """Mirror of ``fast_plan`` (device pointers + capacity)."""

    _fields_ = [("ops", ctypes.c_void_p), ("n_ops", ctypes.c_void_p),
                ("staging_used", ctypes.c_void_p), ("status", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("op_capacity", ctypes.c_int64)]


# (name, restype, argtypes) of every exported entry point; the CPU test
# suite checks that each one is present in the built library.
SIGNATURES: list[tuple[str, object, list]] = [
    ("fast_version", ctypes.c_int, []),
    ("fast_synth_workspace_bytes", ctypes.c_size_t, [ctypes.c_int, ctypes.c_int]),
    ("fast_synth_batch", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
      ctypes.POINTER(FastSchedBufs), ctypes.c_void_p]),
    ("fast_synth_batch_ev", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
      ctypes.POINTER(FastSchedBufs), ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    ("fast_balance_batch", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
      ctypes.POINTER(FastSchedBufs), ctypes.c_void_p]),
    ("fast_decompose_batch", ctypes.c_int,
     [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
      ctypes.POINTER(FastSchedBufs), ctypes.c_void_p]),
    ("fast_compact_workspace_bytes", ctypes.c_size_t, [ctypes.c_int]),
    ("fast_compact_batch", ctypes.c_int,
     [ctypes.POINTER(FastSchedBufs), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
]

_lib: ctypes.CDLL | None = None


def extra_signatures() -> list[tuple[str, object, list]]:
    """Entry points of the executor / MoE front-end (declared lazily so the
    modules that define their structs register them)."""
    from . import _abi_ext

    return _abi_ext.SIGNATURES


def load() -> ctypes.CDLL:
    """Load (building in-tree first if sources are newer) and bind."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("FASTB200_LIB", LIB_PATH)  # experiment builds only
    if path == LIB_PATH and not os.path.exists(LIB_PATH):
        from ._build import build

        build()
    if not os.path.exists(path):
        raise RuntimeError(f"libfastb200.so missing at {path}: run build()")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES + extra_signatures():
        fn = getattr(lib, name, None)
        if fn is None:
            if path != LIB_PATH:  # experiment builds may predate newer entry points
                continue
            raise RuntimeError(f"libfastb200.so lacks symbol {name}")
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check_rc(rc: int, what: str) -> None:
    if rc == FAST_OK:
        return
    from .model import InternalInvariantError, ValidationError

    if rc == FAST_EVALIDATION:
        raise ValidationError(f"{what}: invalid input")
    if rc == FAST_EINVARIANT:
        raise InternalInvariantError(f"{what}: internal invariant broken")
    raise RuntimeError(f"{what}: CUDA error (rc={rc})")
