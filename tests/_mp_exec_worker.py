"""torchrun worker: FastComm (CUDA IPC, one process per GPU) parity.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/_mp_exec_worker.py

Every rank checks its receive buffer against the direct-alltoallv oracle for
several traffic matrices and virtual-server partitions, then checks
all_to_all_fast against NCCL's all_to_all_single on the same tensors.
Exit code 0 only if every rank passed.
"""

from __future__ import annotations

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle.alltoallv import direct_alltoallv, payload  # noqa: E402
from paper_2505_09764_b200 import Topology, workloads  # noqa: E402
from paper_2505_09764_b200.executor import FastComm, all_to_all_fast  # noqa: E402


def partitions(world: int):
    out = []
    for n in range(2, world + 1):
        if world % n == 0:
            out.append((n, world // n))
    return out


def main() -> int:
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    # FAST_MP_ONE_GPU=1: every rank on cuda:0 (a 1-GPU box).  The data path is
    # still the product one -- separate processes, CUDA-IPC mappings of each
    # other's symmetric blocks, system-scope flags -- but NCCL refuses two
    # ranks on one device, so the bootstrap is gloo and the all_to_all_single
    # comparisons use the CPU oracle instead of NCCL.
    one_gpu = os.environ.get("FAST_MP_ONE_GPU") == "1"
    # FAST_MP_GPUS=k: rank r on cuda:(r % k) -- more ranks than GPUs (e.g. the
    # 8-rank 2x4 / 4x2 partitions on a 4-GPU box); gloo bootstrap as above
    share = int(os.environ.get("FAST_MP_GPUS", "0"))
    if share:
        one_gpu = True  # same host-side comparisons (no NCCL with shared devices)
        torch.cuda.set_device(rank % share)
    else:
        torch.cuda.set_device(0 if one_gpu else int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo" if one_gpu else "nccl")
    ok = True
    for (n, m) in partitions(world):
        cases = [workloads.zipf_sizes(5, world, 1.2, 8_000_003),
                 workloads.gen_uniform(6, Topology(n, m), 300_001).sizes,
                 workloads.gen_adversarial(Topology(n, m), 1_234_567).sizes]
        cap = max(int(max(c.sum(0).max(), c.sum(1).max())) for c in cases) + 4096
        cap = max(cap, world * 64 * 4096 * 4 + 4096)  # the all_to_all_fast cases (fp32 rows)
        comm = FastComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20),
                        blocks=16, chunk_bytes=128 * 1024)
        for ci, D in enumerate(cases + cases):
            comm.set_fused(ci < len(cases))  # fused single launch, then multi-launch
            sends_np = [payload(g, int(D[g].sum()) + 16) for g in range(world)]
            send = torch.from_numpy(sends_np[rank]).cuda()
            recv = comm.alltoallv(send, torch.from_numpy(D[rank].copy()).cuda())
            torch.cuda.synchronize()
            comm.check()
            want = direct_alltoallv(sends_np, D)[rank]
            got = recv[: len(want)].cpu().numpy()
            if not np.array_equal(got, want):
                print(f"[rank {rank}] MISMATCH n={n} m={m} case={ci}", flush=True)
                ok = False
            gathered = comm.demand().cpu().numpy()
            if not np.array_equal(gathered, D):
                print(f"[rank {rank}] demand all-gather mismatch", flush=True)
                ok = False
        # graph replays with CHANGING counts in the same device tensor (the
        # config-4 shifting hotspot): the device-side epoch, gather and
        # synthesis must follow the new matrix on every replay
        comm.set_fused(False)
        row_t = torch.zeros(world, dtype=torch.int64, device="cuda")
        for hot in range(3):
            Dh = workloads.gen_hotspot(40 + hot, Topology(n, m), 20_000, hot=hot % world,
                                       factor=8).sizes
            sends_np = [payload(g, int(Dh[g].sum()) + 16) for g in range(world)]
            sbuf = torch.zeros(cap, dtype=torch.uint8, device="cuda")
            sbuf[: sends_np[rank].size].copy_(torch.from_numpy(sends_np[rank]))
            row_t.copy_(torch.from_numpy(Dh[rank].copy()))
            recv = comm.alltoallv(sbuf, row_t)
            torch.cuda.synchronize()
            comm.check()
            want = direct_alltoallv(sends_np, Dh)[rank]
            if not np.array_equal(recv[: len(want)].cpu().numpy(), want):
                print(f"[rank {rank}] graph-replay mismatch n={n} m={m} hot={hot}", flush=True)
                ok = False
        # all_to_all_fast vs NCCL all_to_all_single (rows of 4096 bf16)
        rng = np.random.default_rng(42)
        splits = rng.integers(0, 64, (world, world))
        xs = [torch.randn(int(splits[g].sum()), 4096, dtype=torch.bfloat16,
                          generator=torch.Generator().manual_seed(77 + g)) for g in range(world)]
        x = xs[rank].cuda()
        out_rows = int(splits[:, rank].sum())
        y_fast = torch.empty(out_rows, 4096, dtype=torch.bfloat16, device="cuda")
        all_to_all_fast(y_fast, x, splits[:, rank].tolist(), splits[rank].tolist(), comm=comm)
        if one_gpu:  # all_to_all_single semantics on the host
            y_ref = torch.cat([xs[g][int(splits[g, :rank].sum()):int(splits[g, :rank + 1].sum())]
                               for g in range(world)])
        else:
            y_ref = torch.empty_like(y_fast)
            dist.all_to_all_single(y_ref, x, splits[:, rank].tolist(), splits[rank].tolist())
        torch.cuda.synchronize()
        comm.check()
        if not torch.equal(y_fast.cpu().view(torch.int16), y_ref.cpu().view(torch.int16)):
            print(f"[rank {rank}] all_to_all_fast != all_to_all_single (n={n}, m={m})", flush=True)
            ok = False
        # zero-copy result (a view of the receive region) and the split check
        y0 = all_to_all_fast(None, x, splits[:, rank].tolist(), splits[rank].tolist(), comm=comm)
        torch.cuda.synchronize()
        comm.check()
        if not torch.equal(y0.cpu().view(torch.int16), y_ref.cpu().view(torch.int16)):
            print(f"[rank {rank}] zero-copy all_to_all_fast mismatch (n={n}, m={m})", flush=True)
            ok = False
        # autograd: the backward is the reverse FAST alltoallv (splits swapped)
        from paper_2505_09764_b200.executor import all_to_all_fast_autograd

        xf = xs[rank].float().cuda().requires_grad_(True)
        yf = all_to_all_fast_autograd(xf, splits[:, rank].tolist(), splits[rank].tolist(), comm)
        wg = [torch.randn(int(splits[:, h].sum()), 4096,
                          generator=torch.Generator().manual_seed(900 + h)) for h in range(world)]
        (yf * wg[rank].cuda()).sum().backward()
        torch.cuda.synchronize()
        comm.check()
        # d loss / d x_rank: rows of wg[h] that rank's rows landed on, h-major
        want_g = torch.cat([wg[h][int(splits[:rank, h].sum()):int(splits[:rank + 1, h].sum())]
                            for h in range(world)])
        if not torch.equal(yf.detach().cpu(), y_ref.cpu().float()) or \
                not torch.equal(xf.grad.cpu(), want_g):
            print(f"[rank {rank}] all_to_all_fast autograd mismatch (n={n}, m={m})", flush=True)
            ok = False
        # MoE dispatch (config 3 shape, scaled): expert inputs vs the oracle
        from oracle import moe as moe_oracle
        from paper_2505_09764_b200.moe import MoEDispatch, gating_thresholds

        T, RB = 2048, 8192
        mcomm = FastComm(Topology(n, m), recv_bytes=2 * T * RB * 3, staging_bytes=2 * T * RB * 3,
                         blocks=64)
        disp = MoEDispatch(mcomm, T, RB)
        rngt = np.random.default_rng(500)
        toks = [(rngt.standard_normal((T, RB // 2), dtype=np.float32).view(np.uint32) >> 16)
                .astype(np.uint16).view(np.uint8).reshape(T, RB) for _ in range(world)]
        recv = disp.dispatch(torch.from_numpy(toks[rank]).cuda(), seed=1)
        torch.cuda.synchronize()
        mcomm.check()
        thr, thr2 = gating_thresholds(world)
        topks = [moe_oracle.gate(1, s, T, thr, thr2) for s in range(world)]
        want = moe_oracle.expert_inputs(toks, topks, world)[rank]
        got = recv[: want.size].cpu().numpy().reshape(-1, RB)
        if not np.array_equal(got, want):
            print(f"[rank {rank}] MoE expert input mismatch (n={n}, m={m})", flush=True)
            ok = False
        # fused pack -> send: the executor reads token rows through row_src
        fdisp = MoEDispatch(mcomm, T, RB, fused_pack=True)
        for rep in range(2):  # second call replays the captured graph
            frecv = fdisp.dispatch(torch.from_numpy(toks[rank]).cuda(), seed=1)
            torch.cuda.synchronize()
            mcomm.check()
            if not np.array_equal(frecv[: want.size].cpu().numpy().reshape(-1, RB), want):
                print(f"[rank {rank}] fused-pack MoE expert input mismatch (n={n}, m={m}, "
                      f"call {rep})", flush=True)
                ok = False
        recv = disp.dispatch(torch.from_numpy(toks[rank]).cuda(), seed=1)  # restore disp's state
        torch.cuda.synchronize()
        # combine: experts scale by 2^rank (exact), reverse FAST alltoallv, weighted sum
        n_in = want.size
        expert_out = torch.zeros(2 * T * RB * 3, dtype=torch.uint8, device="cuda")
        xb = (recv[:n_in].view(torch.bfloat16) * (2.0 ** rank)).view(torch.uint8)
        expert_out[:n_in].copy_(xb)
        wts = [np.random.default_rng(900 + s_).random((T, 2), dtype=np.float32) for s_ in range(world)]
        out = torch.empty(T, RB // 2, dtype=torch.bfloat16, device="cuda")
        disp.combine(expert_out, torch.from_numpy(wts[rank]).cuda(), out)
        torch.cuda.synchronize()
        mcomm.check()
        toks16 = [t.view(np.uint16) for t in toks]  # payload bytes read as bf16 (finite: checked)
        finite = all(np.isfinite(moe_oracle.bf16_to_f32(t)).all() for t in toks16)
        if finite:
            wantc = moe_oracle.combine(toks16, topks, wts, lambda e: 2.0 ** e)[rank]
            gotc = out.cpu().view(torch.int16).numpy().view(np.uint16)
            if not np.array_equal(gotc, wantc):
                print(f"[rank {rank}] MoE combine mismatch (n={n}, m={m})", flush=True)
                ok = False
        # router-provided top-k, E = 2 * world experts (2 per rank), k = 2
        E2, L2 = 2 * world, 2
        rdisp = MoEDispatch(mcomm, T, RB, num_experts=E2)
        rtk = [np.random.default_rng(4000 + s_).integers(0, E2, (T, 2)).astype(np.int32)
               for s_ in range(world)]
        rrecv = rdisp.dispatch(torch.from_numpy(toks[rank]).cuda(),
                               topk=torch.from_numpy(rtk[rank]).cuda())
        torch.cuda.synchronize()
        mcomm.check()
        rwant = moe_oracle.expert_inputs(toks, rtk, E2, L2)[rank]
        if not np.array_equal(rrecv[: rwant.size].cpu().numpy().reshape(-1, RB), rwant):
            print(f"[rank {rank}] router-topk MoE expert input mismatch (n={n}, m={m})", flush=True)
            ok = False
        rn = rwant.size
        rexp = torch.zeros(2 * T * RB * 3, dtype=torch.uint8, device="cuda")
        rexp[:rn].copy_((rrecv[:rn].view(torch.bfloat16) * (2.0 ** rank)).view(torch.uint8))
        rout = torch.empty(T, RB // 2, dtype=torch.bfloat16, device="cuda")
        rdisp.combine(rexp, torch.from_numpy(wts[rank]).cuda(), rout)
        torch.cuda.synchronize()
        mcomm.check()
        if finite:
            wantr = moe_oracle.combine(toks16, rtk, wts, lambda e: 2.0 ** (e // L2))[rank]
            if not np.array_equal(rout.cpu().view(torch.int16).numpy().view(np.uint16), wantr):
                print(f"[rank {rank}] router-topk MoE combine mismatch (n={n}, m={m})", flush=True)
                ok = False
        mcomm.close()
        comm.close()
        dist.barrier()
    flag = torch.tensor([0 if ok else 1], device="cpu" if one_gpu else "cuda")
    dist.all_reduce(flag)
    if rank == 0:
        print("MP_EXEC", "PASS" if int(flag.item()) == 0 else "FAIL", flush=True)
    dist.destroy_process_group()
    return 0 if int(flag.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
