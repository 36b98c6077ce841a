"""CPU ORACLE -- test infrastructure only, never the product path.

ctypes front-end of oracle/fast_oracle.c, the plain-C restatement of the
reference scheduler (tiersched.synthesize_fast, pipeline.py:52-59).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this
module.  Parity of the restatement is pinned against the reference itself by
tests/test_oracle.py (golden fixtures made by tests/golden/make_golden.py
from tiersched, plus a live comparison when /root/reference is present).

Outputs are dicts of numpy arrays named like the fields of
``paper_2505_09764_b200.schedule.PackedSchedule``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libfastoracle.so")

MOVE_DTYPE = np.dtype([("bytes", "<i8"), ("from_gpu", "<i4"), ("to_gpu", "<i4")])

_lib = None


def build() -> str:
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        src = os.path.join(HERE, "fast_oracle.c")
        if not os.path.exists(LIB) or os.path.getmtime(src) > os.path.getmtime(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def stage_cap(n: int) -> int:
    return n * n - 2 * n + 2


def synthesize_batch(D: np.ndarray, n: int, m: int) -> dict:
    """Oracle synthesize_fast for D of shape [B,G,G] (or [G,G])."""
    D = np.ascontiguousarray(D, dtype=np.int64)
    single = D.ndim == 2
    if single:
        D = D[None]
    B, G = D.shape[0], n * m
    assert D.shape[1:] == (G, G)
    T, S, K = n * (n - 1), max(m - 1, 1), stage_cap(n)
    out = dict(
        balanced=np.zeros((B, G, G), np.int64), server=np.zeros((B, n, n), np.int64),
        move_count=np.zeros((B, T), np.int32), moves=np.zeros((B, T, S), MOVE_DTYPE),
        common_sum=np.zeros(B, np.int64), aux=np.zeros((B, n, n), np.int64),
        n_raw=np.zeros(B, np.int32), stage_weight=np.zeros((B, K), np.int64),
        stage_perm=np.zeros((B, K, n), np.uint8), stage_bytes=np.zeros((B, K, n), np.int64),
        n_stages=np.zeros(B, np.int32), stage_order=np.zeros((B, K), np.int32),
        status=np.zeros(B, np.int32))
    lib = _load()
    lib.fo_synthesize_batch(
        ctypes.c_int(B), ctypes.c_int(n), ctypes.c_int(m), _p(D), _p(out["balanced"]),
        _p(out["server"]), _p(out["move_count"]), _p(out["moves"]), _p(out["common_sum"]),
        _p(out["aux"]), _p(out["n_raw"]), _p(out["stage_weight"]), _p(out["stage_perm"]),
        _p(out["stage_bytes"]), _p(out["n_stages"]), _p(out["stage_order"]), _p(out["status"]))
    return out


def dfs_counters(reset: bool = True) -> tuple[int, int]:
    """(DFS steps, searches) accumulated by the oracle since the last reset
    (one step = one column newly marked seen in the Kuhn search)."""
    lib = _load()
    lib.fo_dfs_counters.restype = ctypes.c_int64
    s = ctypes.c_int64()
    steps = lib.fo_dfs_counters(ctypes.byref(s), ctypes.c_int(1 if reset else 0))
    return int(steps), int(s.value)


def decompose_server(S: np.ndarray) -> dict:
    """Oracle decompose_server_matrix + strip + sort for one n x n matrix."""
    S = np.ascontiguousarray(S, dtype=np.int64)
    n = S.shape[0]
    K = stage_cap(n)
    out = dict(common_sum=np.zeros(1, np.int64), aux=np.zeros((n, n), np.int64),
               n_raw=np.zeros(1, np.int32), stage_weight=np.zeros(K, np.int64),
               stage_perm=np.zeros((K, n), np.uint8), stage_bytes=np.zeros((K, n), np.int64),
               n_stages=np.zeros(1, np.int32), stage_order=np.zeros(K, np.int32))
    st = _load().fo_decompose_server(
        ctypes.c_int(n), _p(S), _p(out["common_sum"]), _p(out["aux"]), _p(out["n_raw"]),
        _p(out["stage_weight"]), _p(out["stage_perm"]), _p(out["stage_bytes"]),
        _p(out["n_stages"]), _p(out["stage_order"]))
    out["status"] = int(st)
    return out


def packed_fields(out: dict, b: int, n: int, m: int) -> dict:
    """Per-matrix kwargs for PackedSchedule (trimmed to the used lengths)."""
    k = int(out["n_raw"][b])
    s = int(out["n_stages"][b])
    return dict(
        n=n, m=m, status=int(out["status"][b]), balanced=out["balanced"][b],
        server=out["server"][b], move_count=out["move_count"][b], moves=out["moves"][b],
        common_sum=int(out["common_sum"][b]), aux=out["aux"][b], n_raw=k,
        stage_weight=out["stage_weight"][b][:k], stage_perm=out["stage_perm"][b][:k],
        stage_bytes=out["stage_bytes"][b][:k], n_stages=s,
        stage_order=out["stage_order"][b][:s])
