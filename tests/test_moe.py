"""MoE dispatch front-end (BASELINE config 3): gating -> histogram/scan ->
pack -> FAST alltoallv -> unpack, against the numpy oracle (oracle/moe.py).

CPU part: the oracle's invariants and the product's thresholds.  GPU part:
all 8 ranks of a 2x4 partition on one B200 (group mode): topk, counts,
send buffer and every GPU's expert input are byte-identical to the oracle.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from oracle import moe as moe_oracle
from oracle.alltoallv import payload
from paper_2505_09764_b200.moe import gating_thresholds


def test_thresholds_match_oracle_and_exclude_first_choice():
    for E, hot in [(8, 0), (8, 5), (4, 1), (16, 3)]:
        thr, thr2 = gating_thresholds(E, 0.8, hot)
        othr, othr2 = moe_oracle.thresholds(E, 0.8, hot)
        assert np.array_equal(thr, othr) and np.array_equal(thr2, othr2)
        topk = moe_oracle.gate(7, 1, 5000, thr, thr2)
        assert (topk[:, 0] != topk[:, 1]).all()
        assert topk.min() >= 0 and topk.max() < E
        counts = np.bincount(topk[:, 0], minlength=E)
        assert counts[hot] == counts.max()  # the hot expert is the most popular


@pytest.mark.gpu
def test_moe_dispatch_group_mode_matches_oracle():
    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.executor import GroupComm, GroupRank
    from paper_2505_09764_b200.moe import MoEDispatch

    G, T, RB, seed = 8, 3000, 1024, 2
    tokens_np = [payload(100 + s, T * RB).reshape(T, RB) for s in range(G)]
    cap = 2 * T * RB * 4
    group = GroupComm(Topology(2, 4), recv_bytes=cap, staging_bytes=cap, blocks=8)
    thr, thr2 = gating_thresholds(G)
    disps, rows = [], []
    for s in range(G):
        d = MoEDispatch(GroupRank(group, s), T, RB)
        d.route(seed)
        d.pack(torch.from_numpy(tokens_np[s]).cuda())
        disps.append(d)
        rows.append(d.demand_row)
    torch.cuda.synchronize()
    topks = []
    for s, d in enumerate(disps):
        want = moe_oracle.gate(seed, s, T, thr, thr2)
        got = d.topk.cpu().numpy().reshape(T, 2)
        assert np.array_equal(got, want), s
        topks.append(want)
        counts, seg, _ = moe_oracle.route(want, G)
        assert np.array_equal(d.counts.cpu().numpy(), counts)
        assert np.array_equal(d.seg_rows.cpu().numpy(), seg)
        send = d.send[: 2 * T * RB].cpu().numpy().reshape(2 * T, RB)
        assert np.array_equal(send, moe_oracle.pack(tokens_np[s], want, G)), s
    Dfull = torch.stack(rows)
    selfb = torch.diagonal(Dfull).clone()
    D = Dfull.clone()
    D.fill_diagonal_(0)
    recvs = group.alltoallv([d.send for d in disps], D, self_bytes=selfb)
    for s, d in enumerate(disps):
        d.unpack(D=D, self_sizes=selfb, recv=recvs[s])
    torch.cuda.synchronize()
    group.check()
    want = moe_oracle.expert_inputs(tokens_np, topks, G)
    for h in range(G):
        n = want[h].shape[0] * RB
        got = recvs[h][:n].cpu().numpy().reshape(-1, RB)
        assert np.array_equal(got, want[h]), h
    # fused pack -> send: no send buffer; the executor reads token rows
    # through row_src (fast_comm_set_send_rows), same expert inputs
    for r in recvs:
        r.fill_(0xA5)
    fdisps, srows, toks_dev = [], [], []
    for s in range(G):
        d = MoEDispatch(GroupRank(group, s), T, RB, fused_pack=True)
        tk = torch.from_numpy(tokens_np[s]).cuda()
        d.route(seed)
        d.rowmap(tokens=tk)
        fdisps.append(d)
        toks_dev.append(tk)
        srows.append((d._tokens, d.row_src, RB))
    torch.cuda.synchronize()
    for s, d in enumerate(fdisps):
        _, seg, _ = moe_oracle.route(topks[s], G)
        packed = moe_oracle.pack(tokens_np[s], topks[s], G)
        rs = d.row_src.cpu().numpy()
        assert np.array_equal(tokens_np[s][rs], packed), s  # row map == pack order
    recvs = group.alltoallv([t.view(torch.uint8).reshape(-1) for t in toks_dev], D,
                            self_bytes=selfb, send_rows=srows)
    for s, d in enumerate(fdisps):
        d.unpack(D=D, self_sizes=selfb, recv=recvs[s])
    torch.cuda.synchronize()
    group.check()
    for h in range(G):
        n = want[h].shape[0] * RB
        got = recvs[h][:n].cpu().numpy().reshape(-1, RB)
        assert np.array_equal(got, want[h]), ("fused", h)
    group.close()


@pytest.mark.gpu
@pytest.mark.parametrize("RB", [48, 1040, 4112])
def test_fused_pack_odd_row_sizes_group_mode(RB):
    """Row-mapped send with row_bytes not a power of two (the executor's
    u32 magic division) and FAST's byte-granular splits crossing rows: the
    fused and the packed dispatch give identical expert inputs."""
    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.executor import GroupComm, GroupRank
    from paper_2505_09764_b200.moe import MoEDispatch

    G, T, seed = 4, 1500, 9
    toks = [torch.from_numpy(payload(300 + s, T * RB).reshape(T, RB)).cuda() for s in range(G)]
    cap = 2 * T * RB * 4
    outs = {}
    for fused in (False, True):
        group = GroupComm(Topology(2, 2), recv_bytes=cap, staging_bytes=cap, blocks=8,
                          chunk_bytes=4096 + 16 * 3)
        ds = [MoEDispatch(GroupRank(group, s), T, RB, fused_pack=fused) for s in range(G)]
        for s, d in enumerate(ds):
            d.route(seed)
            d.rowmap(tokens=toks[s]) if fused else d.pack(toks[s])
        Dfull = torch.stack([d.demand_row for d in ds])
        selfb = torch.diagonal(Dfull).clone()
        D = Dfull.clone()
        D.fill_diagonal_(0)
        sends = [t.view(torch.uint8).reshape(-1) for t in toks] if fused else [d.send for d in ds]
        rows = [(d._tokens, d.row_src, RB) for d in ds] if fused else None
        recvs = group.alltoallv(sends, D, self_bytes=selfb, send_rows=rows)
        for s, d in enumerate(ds):
            d.unpack(D=D, self_sizes=selfb, recv=recvs[s])
        torch.cuda.synchronize()
        group.check()
        outs[fused] = [recvs[h][: int(Dfull[:, h].sum())].cpu().numpy() for h in range(G)]
        group.close()
    for h in range(G):
        assert np.array_equal(outs[True][h], outs[False][h]), h


@pytest.mark.gpu
def test_moe_combine_group_mode_matches_oracle():
    """dispatch -> experts (x * 2^e, exact) -> reverse FAST alltoallv (D^T) ->
    weighted combine: bit-exact vs the numpy oracle."""
    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.executor import GroupComm, GroupRank
    from paper_2505_09764_b200.moe import MoEDispatch

    G, T, H, seed = 8, 2000, 512, 4
    RB = 2 * H
    gen = torch.Generator().manual_seed(0)
    toks = [torch.randn(T, H, generator=gen).to(torch.bfloat16) for _ in range(G)]
    toks_u16 = [t.view(torch.int16).numpy().view(np.uint16) for t in toks]
    weights = [torch.rand(T, 2, generator=gen, dtype=torch.float32) for _ in range(G)]
    cap = 2 * T * RB * 4
    group = GroupComm(Topology(2, 4), recv_bytes=cap, staging_bytes=cap, blocks=8)
    disps = []
    for s in range(G):
        d = MoEDispatch(GroupRank(group, s), T, RB)
        d.route(seed)
        d.pack(toks[s].cuda())
        disps.append(d)
    Dfull = torch.stack([d.demand_row for d in disps])
    selfb = torch.diagonal(Dfull).clone()
    D = Dfull.clone()
    D.fill_diagonal_(0)
    recvs = group.alltoallv([d.send for d in disps], D, self_bytes=selfb)
    expert_out = []
    for h, d in enumerate(disps):
        d.unpack(D=D, self_sizes=selfb, recv=recvs[h])
        d.remember_forward(D, selfb)
        n_in = int(Dfull[:, h].sum().item())
        x = recvs[h][:n_in].view(torch.bfloat16) * (2.0 ** h)  # expert h (exact)
        buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
        buf[:n_in].copy_(x.view(torch.uint8))
        expert_out.append(buf)
    # reverse alltoallv: rank h sends column h of the forward D back (D^T)
    Dt = D.t().contiguous()
    comb = group.alltoallv(expert_out, Dt, self_bytes=selfb)
    outs = []
    for s, d in enumerate(disps):
        o = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
        d.combine_rows(comb[s], expert_out[s], weights[s].cuda(), o)
        outs.append(o)
    torch.cuda.synchronize()
    group.check()
    thr, thr2 = gating_thresholds(G)
    topks = [moe_oracle.gate(seed, s, T, thr, thr2) for s in range(G)]
    want = moe_oracle.combine(toks_u16, topks, [w.numpy() for w in weights], lambda e: 2.0 ** e)
    for s in range(G):
        got = outs[s].cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, want[s]), s
    group.close()


@pytest.mark.gpu
@pytest.mark.parametrize("k,L", [(1, 2), (4, 2), (2, 3)])
def test_router_topk_experts_per_rank_group_mode(k, L):
    """The router's top-k ids (any k in 1/2/4/8, duplicates allowed) with
    E = L * world experts, L per rank: expert inputs and the weighted
    combine are bit-exact vs the numpy oracle (group mode, 2x2)."""
    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.executor import GroupComm, GroupRank
    from paper_2505_09764_b200.moe import MoEDispatch

    G, T, H = 4, 1200, 256
    E = G * L
    RB = 2 * H
    gen = torch.Generator().manual_seed(k * 10 + L)
    toks = [torch.randn(T, H, generator=gen).to(torch.bfloat16) for _ in range(G)]
    toks_u8 = [t.view(torch.uint8).numpy().reshape(T, RB) for t in toks]
    toks_u16 = [t.view(torch.int16).numpy().view(np.uint16) for t in toks]
    topks = [np.random.default_rng(70 + s).integers(0, E, (T, k)).astype(np.int32)
             for s in range(G)]
    weights = [torch.rand(T, k, generator=gen, dtype=torch.float32) for _ in range(G)]
    cap = k * T * RB * 4
    group = GroupComm(Topology(2, 2), recv_bytes=cap, staging_bytes=cap, blocks=8)
    ds = []
    for s in range(G):
        d = MoEDispatch(GroupRank(group, s), T, RB, k=k, num_experts=E)
        d.route(topk=torch.from_numpy(topks[s]).cuda())
        d.pack(toks[s].cuda())
        ds.append(d)
    torch.cuda.synchronize()
    for s, d in enumerate(ds):
        counts, _, _ = moe_oracle.route(topks[s], E)
        assert np.array_equal(d.counts.cpu().numpy(), counts), s
        dr = d.demand_row.cpu().numpy()
        assert np.array_equal(dr, counts.reshape(G, L).sum(1) * RB), s
    Dfull = torch.stack([d.demand_row for d in ds])
    selfb = torch.diagonal(Dfull).clone()
    D = Dfull.clone()
    D.fill_diagonal_(0)
    recvs = group.alltoallv([d.send for d in ds], D, self_bytes=selfb)
    for s, d in enumerate(ds):
        d.unpack(D=D, self_sizes=selfb, recv=recvs[s])
    torch.cuda.synchronize()
    group.check()
    want = moe_oracle.expert_inputs(toks_u8, topks, E, L)
    expert_out = []
    for h, d in enumerate(ds):
        n_in = want[h].size
        assert np.array_equal(recvs[h][:n_in].cpu().numpy().reshape(-1, RB), want[h]), h
        d.remember_forward(D, selfb)
        x = recvs[h][:n_in].view(torch.bfloat16) * (2.0 ** h)  # rank h's experts (exact)
        buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
        buf[:n_in].copy_(x.view(torch.uint8))
        expert_out.append(buf)
    comb = group.alltoallv(expert_out, D.t().contiguous(), self_bytes=selfb)
    outs = []
    for s, d in enumerate(ds):
        o = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
        d.combine_rows(comb[s], expert_out[s], weights[s].cuda(), o)
        outs.append(o)
    torch.cuda.synchronize()
    group.check()
    wantc = moe_oracle.combine(toks_u16, topks, [w.numpy() for w in weights],
                               lambda e: 2.0 ** (e // L))
    for s in range(G):
        assert np.array_equal(outs[s].cpu().view(torch.int16).numpy().view(np.uint16),
                              wantc[s]), s
    group.close()


@pytest.mark.gpu
def test_router_topk_invalid_ids_fail_loudly():
    """An expert id outside [0, E) poisons the demand row (-1): the
    alltoallv's synthesis rejects the matrix instead of dropping tokens."""
    from paper_2505_09764_b200 import Topology
    from paper_2505_09764_b200.executor import GroupComm, GroupRank
    from paper_2505_09764_b200.moe import MoEDispatch

    group = GroupComm(Topology(2, 1), recv_bytes=1 << 20, staging_bytes=1 << 20, blocks=4)
    d = MoEDispatch(GroupRank(group, 0), 64, 256, k=2, num_experts=4)
    tk = np.random.default_rng(0).integers(0, 4, (64, 2)).astype(np.int32)
    tk[5, 1] = 9
    d.route(topk=torch.from_numpy(tk).cuda())
    assert (d.demand_row.cpu().numpy() == -1).all()
    group.close()
