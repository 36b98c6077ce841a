"""Executor flag protocol under randomised delays (protocol
stress).  libfastb200_fuzz.so is the product library built with
-DFAST_EXEC_FUZZ: every signal (red/st.release.sys) and every wait
(ld.acquire spin) is preceded by a pseudo-random 0-4 us sleep, so producers,
forwarders and consumers interleave in orders the plain build rarely shows.
The group-mode executor parity tests and the 1-GPU multi-process IPC worker
run against it in subprocesses (FASTB200_LIB selects the library)."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest
import torch

from conftest import REPO

pytestmark = pytest.mark.gpu

FUZZ_LIB = os.path.join(REPO, "paper_2505_09764_b200", "libfastb200_fuzz.so")


def _fuzz_lib() -> str:
    if not os.path.exists(FUZZ_LIB):
        sys.path.insert(0, REPO)
        from paper_2505_09764_b200 import _build

        _build.build(force=True, extra=["-DFAST_EXEC_FUZZ"], out=FUZZ_LIB)
    return FUZZ_LIB


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_group_executor_parity_under_fuzz():
    env = dict(os.environ, FASTB200_LIB=_fuzz_lib())
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        os.path.join(REPO, "tests", "test_exec_gpu.py"), "-k",
                        "matches_direct or config2 or edge_cases or wide or small_buffers"],
                       capture_output=True, text=True, timeout=1200, cwd=REPO, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_multiprocess_ipc_under_fuzz():
    env = dict(os.environ, FASTB200_LIB=_fuzz_lib(), FAST_MP_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(REPO, "tests", "_mp_exec_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=REPO, env=env)
    assert r.returncode == 0 and "MP_EXEC PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
