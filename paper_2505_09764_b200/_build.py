"""In-tree build of libfastb200.so (sm_100a) with nvcc.

The shared library is the product: every CUDA kernel of the hot path plus the
C-ABI declared in include/fastb200.h.  It is built next to this file so that
it travels with the repo snapshot to the GPU box (``*.so`` is git-ignored).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO_DIR, "include")
LIB_PATH = os.path.join(PKG_DIR, "libfastb200.so")

SOURCES = ["synth.cu", "exec.cu", "moe.cu", "sim.cu", "stages.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--cudart", "static",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libfastb200.so")


def sources() -> list[str]:
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def needs_build() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    lib_m = os.path.getmtime(LIB_PATH)
    deps = sources() + [os.path.join(INCLUDE, "fastb200.h")]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    return any(os.path.getmtime(p) > lib_m for p in deps)


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          out: str | None = None) -> str:
    """Compile each translation unit in parallel (nvcc -c), then link the
    shared library.  `extra` flags (e.g. -DFAST_EXEC_FUZZ) and `out` build a
    variant library next to the product one."""
    out = out or LIB_PATH
    if not force and out == LIB_PATH and not needs_build():
        return LIB_PATH
    nvcc = _nvcc()
    objdir = os.path.join(PKG_DIR, "_obj", os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    comp = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra or [])
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *comp, f"-I{INCLUDE}", f"-I{CSRC}", "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    bad = [p.args[-1] for p in procs if p.wait() != 0]
    if bad:
        raise RuntimeError(f"nvcc failed on {bad}")
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "--cudart", "static",
            "-o", out + ".tmp", *objs]
    subprocess.run(link, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
