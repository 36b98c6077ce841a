"""The C-ABI library loads and exports every symbol include/*.h declares.

CPU-only: no compute calls (there is no GPU in the build container).
"""

from __future__ import annotations

import ctypes
import os
import re

from conftest import REPO
from paper_2505_09764_b200 import _lib


def declared_functions() -> set[str]:
    names = set()
    inc = os.path.join(REPO, "include")
    for f in os.listdir(inc):
        if not f.endswith(".h"):
            continue
        text = open(os.path.join(inc, f)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:int|size_t|void|const char\s*\*)\s+\**(fast_\w+)\s*\(",
                             text, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = declared_functions()
    assert {"fast_synth_batch", "fast_balance_batch", "fast_decompose_batch"} <= decl
    raw = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(decl) if not hasattr(raw, n)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES + _lib.extra_signatures()}
    assert decl <= bound, sorted(decl - bound)
    assert lib.fast_version() >= 100


def test_workspace_sizing_is_host_only():
    lib = _lib.load()
    assert lib.fast_synth_workspace_bytes(0, 8) == 0
    assert lib.fast_synth_workspace_bytes(10, 0) == 0
    assert lib.fast_synth_workspace_bytes(10, 1) == 10 * 256  # 1 x 1 decompose inputs
    assert lib.fast_synth_workspace_bytes(10, 129) == 0
    assert lib.fast_synth_workspace_bytes(1000, 128) > 1000 * 2 * 128 * 128 * 8


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2505_09764_b200 import Topology, gen_uniform, synthesize_fast

    with pytest.raises(RuntimeError, match="CUDA"):
        synthesize_fast(gen_uniform(0, Topology(2, 2), 10), Topology(2, 2))
