"""Multi-process FastComm over CUDA IPC: one process per rank, each rank maps
its peers' symmetric blocks with cudaIpcOpenMemHandle and synchronises with
system-scope flags (the paper's runtime).

With >= 2 GPUs the ranks sit on distinct GPUs (P2P over NVSwitch, NCCL as the
comparison bar).  On a 1-GPU box the same worker runs with every rank on
cuda:0 (FAST_MP_ONE_GPU=1): the processes are still separate CUDA contexts
that reach each other only through IPC mappings and system-scope flags, so the
IPC open, the cross-process flag protocol, the fused single-launch path and
all_to_all_fast are exercised; the contexts time-slice, so the cases are small
and the executor's spins are bounded (a hang becomes status 3, not a stall).
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest
import torch

from conftest import REPO

pytestmark = pytest.mark.gpu


def _run(nproc: int, env_extra: dict, port: int) -> None:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(REPO, "tests", "_mp_exec_worker.py")]
    env = dict(os.environ, **env_extra)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP_EXEC PASS" in r.stdout


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_fastcomm_multiprocess_parity():
    _run(min(8, torch.cuda.device_count()), {}, 29533)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
@pytest.mark.parametrize("nproc", [2, 4])
def test_fastcomm_multiprocess_one_gpu(nproc):
    """Separate processes on ONE device: IPC mappings + system-scope flags."""
    _run(nproc, {"FAST_MP_ONE_GPU": "1"}, 29540 + nproc)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_fastcomm_eight_ranks_shared_gpus():
    """8 ranks (the 2x4 and 4x2 partitions of BASELINE configs 2-4) on the
    GPUs available, two or more processes per device: cross-GPU IPC
    mappings and same-GPU ones in one communicator."""
    _run(8, {"FAST_MP_GPUS": str(min(4, torch.cuda.device_count()))}, 29560)
