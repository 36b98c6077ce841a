"""Host-side logic of the multi-GPU path on CPU (gloo): world_size 2 (2x1)
and world_size 8 in the two partitions the 8-GPU runs use (2x4, 4x2).

* count all-gather semantics: every rank assembles the same D (zero
  diagonal) and self-size vector from the per-rank rows;
* every rank independently derives the identical schedule and plan from
  the gathered D (the paper's "same schedule on every GPU, no exchange",
  PAPER.md:615);
* message-passing execution of the plan: each rank runs only its own ops
  phase by phase and ships the written bytes to their owners; every
  receive buffer equals the direct alltoallv (self slot left as a gap);
* all_to_all_fast's split/offset arithmetic against gloo's
  all_to_all_single, with a stand-in transport.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO



def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _GlooComm:
    """Stand-in transport with FastComm's alltoallv contract (receive layout
    of all_to_all_single with a gap at the self slot)."""

    recv_bytes = 1 << 30

    def __init__(self):
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.split_errors = 0

    def _counts_for(self, splits, row_bytes, out=False):
        return torch.tensor([int(x) * int(row_bytes) for x in splits], dtype=torch.int64)

    def _check_output_splits(self, out_bytes):
        col = self.D[:, self.rank]
        self.split_errors += int((col != out_bytes).any())

    def alltoallv(self, send: torch.Tensor, counts: torch.Tensor,
                  copy_self: bool = False) -> torch.Tensor:
        rows = [torch.zeros(self.world, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(rows, counts.to(torch.int64))
        D = torch.stack(rows)
        self.D = D
        out_splits = D[:, self.rank].tolist()
        recv = torch.zeros(int(sum(out_splits)) + 4096, dtype=torch.uint8)  # region slack
        dist.all_to_all_single(recv[: int(sum(out_splits))], send[: int(counts.sum())], out_splits,
                               counts.tolist())
        lo = int(sum(out_splits[: self.rank]))
        if not copy_self:
            recv[lo:lo + out_splits[self.rank]] = 0  # the self slot is a gap
        return recv


def _worker(rank: int, port: int, errq, WORLD: int, n: int, m: int):
    import sys

    sys.path.insert(0, REPO)
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from oracle import oracle
        from oracle.alltoallv import direct_alltoallv, payload
        from paper_2505_09764_b200 import workloads
        from paper_2505_09764_b200.executor import (BUF_RECV, BUF_SEND, all_to_all_fast,
                                                    plan_compile_host)
        from paper_2505_09764_b200.schedule import PackedSchedule

        G = n * m
        assert G == WORLD
        D = workloads.zipf_sizes(11, G, 1.2, 200_003 * G)
        selfb = np.array([777 + 457 * g for g in range(G)], dtype=np.int64)
        Dfull = D + np.diag(selfb)
        # 1. count all-gather (mirrors gather_demand_kernel's layout)
        rows = [torch.zeros(G, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(rows, torch.from_numpy(Dfull[rank].copy()))
        Dg = torch.stack(rows).numpy()
        D0 = Dg.copy()
        np.fill_diagonal(D0, 0)
        assert np.array_equal(D0, D) and np.array_equal(np.diagonal(Dg), selfb)
        # 2. schedule + plan on every rank, identical everywhere
        out = oracle.synthesize_batch(D0, n, m)
        p = PackedSchedule(**oracle.packed_fields(out, 0, n, m))
        cap = int(Dfull.sum(axis=0).max()) + 64
        ops, _, st = plan_compile_host(D0, n, m, p.stage_order, p.stage_perm, p.stage_bytes,
                                       cap, cap, send_self=selfb, chunk=4096)
        assert st == 0
        allops = [None] * G
        dist.all_gather_object(allops, ops.tobytes())
        assert all(x == allops[0] for x in allops)
        # 3. message passing: each rank executes only its own ops, per phase
        send = payload(rank, int(Dfull[rank].sum()))
        recv = np.zeros(cap, np.uint8)
        stg = np.zeros(cap + 64, np.uint8)
        for ph in range(4):
            msgs = []
            for o in ops[(ops["phase"] == ph) & (ops["exec_rank"] == rank)]:
                src = send if o["src_buf"] == BUF_SEND else stg
                so, ln = int(o["src_off"]), int(o["len"])
                msgs.append((int(o["dst_rank"]), int(o["dst_buf"]), int(o["dst_off"]),
                             src[so:so + ln].tobytes()))
            got = [None] * G
            dist.all_gather_object(got, msgs)
            for lst in got:
                for dst, buf, off, data in lst:
                    if dst != rank:
                        continue
                    arr = np.frombuffer(data, np.uint8)
                    (recv if buf == BUF_RECV else stg)[off:off + len(arr)] = arr
        full = direct_alltoallv([payload(g, int(Dfull[g].sum())) for g in range(G)], Dfull)[rank]
        lo = int(Dfull[:rank, rank].sum())
        hi = lo + int(selfb[rank])
        assert np.array_equal(recv[:lo], full[:lo])
        assert np.array_equal(recv[hi:len(full)], full[hi:])
        # 4. all_to_all_fast offset arithmetic vs all_to_all_single
        splits = np.random.default_rng(5).integers(0, 7, (G, G))
        x = torch.arange(int(splits[rank].sum()) * 6, dtype=torch.int32).reshape(-1, 6) + 1000 * rank
        y_fast = torch.zeros(int(splits[:, rank].sum()), 6, dtype=torch.int32)
        y_ref = torch.zeros_like(y_fast)
        gc = _GlooComm()
        all_to_all_fast(y_fast, x, splits[:, rank].tolist(), splits[rank].tolist(), comm=gc)
        dist.all_to_all_single(y_ref, x, splits[:, rank].tolist(), splits[rank].tolist())
        assert torch.equal(y_fast, y_ref)
        y0 = all_to_all_fast(None, x, splits[:, rank].tolist(), splits[rank].tolist(), comm=gc)
        assert torch.equal(y0, y_ref) and gc.split_errors == 0  # zero-copy view
        wrong = splits[:, rank].copy()
        wrong[(rank + 1) % G] += 1
        all_to_all_fast(None, x, wrong.tolist(), splits[rank].tolist(), comm=gc)
        assert gc.split_errors == 1  # output splits checked against the gathered counts
        # 5. autograd: backward is the reverse alltoallv (splits swapped)
        from paper_2505_09764_b200.executor import all_to_all_fast_autograd

        xf = (x.to(torch.float64) / 7).requires_grad_(True)
        yf = all_to_all_fast_autograd(xf, splits[:, rank].tolist(), splits[rank].tolist(), gc)
        wgt = torch.arange(yf.numel(), dtype=torch.float64).reshape(yf.shape) + rank
        (yf * wgt).sum().backward()
        want = torch.zeros_like(xf)
        dist.all_to_all_single(want, wgt, splits[rank].tolist(), splits[:, rank].tolist())
        assert torch.equal(xf.grad, want)
        dist.destroy_process_group()
    except Exception as exc:  # pragma: no cover - reported by the parent
        import traceback

        errq.put(f"rank {rank}: {exc!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,n,m", [(2, 2, 1), (8, 2, 4), (8, 4, 2)])
def test_multi_rank_host_logic_gloo(world, n, m):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, errq, world, n, m))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
