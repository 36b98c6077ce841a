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
    group.close()
