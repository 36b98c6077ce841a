"""Small invocations of every product kernel, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py

Covers: balance / decompose / sort / strip-table / compact (fast_synth_batch,
fast_compact_batch), the standalone match and strip+sort kernels, the device
plan compile, the group-mode executor (all ranks in one cooperative launch,
plain and row-mapped sends), the MoE gate / route / pack / rowmap / unpack /
combine kernels and the analytical model.  Every result is also checked
against the CPU oracle, so a sanitizer run is a parity run too.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import oracle
from oracle.alltoallv import direct_alltoallv, payload
from paper_2505_09764_b200 import Topology, schedule_to_json, synth, workloads
from paper_2505_09764_b200.executor import GroupComm, GroupRank
from paper_2505_09764_b200.moe import MoEDispatch

torch.cuda.set_device(0)
done = []

# synthesis, full and compact layouts, several shapes (incl. n > 32: global work matrix)
for n, m, B in [(2, 4, 3), (4, 2, 3), (5, 3, 2), (40, 8, 2)]:
    D = np.stack([workloads.zipf_sizes(b, n * m, 0.9, 10**8) for b in range(B)])
    ref = oracle.synthesize_batch(D, n, m)
    p = synth.synthesize_packed(torch.from_numpy(D).cuda(), n, m).host()
    hs = synth.synthesize_host_batch(torch.from_numpy(D).pin_memory(), n, m, chunk=2)
    for b in range(B):
        want = oracle.packed_fields(ref, b, n, m)
        assert np.array_equal(p[b].balanced, want["balanced"])
        assert np.array_equal(hs.packed(b, D[b]).stage_bytes, want["stage_bytes"])
done.append("synthesis (balance, decompose, sort, strip table, compact)")

# standalone building blocks
from paper_2505_09764_b200 import ServerMatrix  # noqa: E402

S = np.array([[0, 5, 3], [1, 0, 4], [6, 2, 0]], np.int64)
dec = synth.decompose_server_matrix(ServerMatrix(S))
st = synth.sort_stages_ascending(synth.strip_auxiliary(dec.stages, dec.aux))
assert synth.find_perfect_matching(np.ones((4, 4))) == {0: 3, 1: 2, 2: 1, 3: 0}
done.append("match / strip+sort kernels")

# executor, group mode (plan compile + exec), plain and row-mapped sends
for n, m in [(2, 2), (2, 4), (4, 2)]:
    G = n * m
    Dm = workloads.zipf_sizes(3, G, 1.2, 1 << 20)
    cap = int(max(Dm.sum(0).max(), Dm.sum(1).max())) + 4096
    comm = GroupComm(Topology(n, m), recv_bytes=cap, staging_bytes=2 * cap + (1 << 20), blocks=4,
                     chunk_bytes=64 * 1024)
    sends_np = [payload(g, int(Dm[g].sum()) + 16) for g in range(G)]
    recvs = comm.alltoallv([torch.from_numpy(x).cuda() for x in sends_np],
                           torch.from_numpy(Dm).cuda())
    torch.cuda.synchronize()
    comm.check()
    want = direct_alltoallv(sends_np, Dm)
    for h in range(G):
        assert np.array_equal(recvs[h][: len(want[h])].cpu().numpy(), want[h])
    comm.close()
done.append("plan compile + group-mode exec")

# MoE front-end on a 2x2 group (gate, route, pack, unpack, rowmap, combine)
from oracle import moe as moe_oracle  # noqa: E402

G, T, RB = 4, 512, 256
group = GroupComm(Topology(2, 2), recv_bytes=2 * T * RB * 3, staging_bytes=2 * T * RB * 3,
                  blocks=4)
toks = [payload(50 + s, T * RB).reshape(T, RB) for s in range(G)]
ds = []
for s in range(G):
    d = MoEDispatch(GroupRank(group, s), T, RB)
    d.route(1)
    d.pack(torch.from_numpy(toks[s]).cuda())
    d.rowmap(tokens=torch.from_numpy(toks[s]).cuda())
    ds.append(d)
Dm = torch.stack([d.demand_row for d in ds]).clone()
selfb = torch.diagonal(Dm).clone()
Dm.fill_diagonal_(0)
group.alltoallv([d.send for d in ds], Dm, self_bytes=selfb)
for s, d in enumerate(ds):
    d.unpack(D=Dm.contiguous(), self_sizes=selfb, recv=group.recvs[s])
torch.cuda.synchronize()
group.check()
thr, thr2 = moe_oracle.thresholds(G)
topks = [moe_oracle.gate(1, s, T, thr, thr2) for s in range(G)]
want = moe_oracle.expert_inputs(toks, topks, G)
for s in range(G):
    assert np.array_equal(group.recvs[s][: want[s].size].cpu().numpy().reshape(-1, RB), want[s])
done.append("MoE gate / route / pack / rowmap / unpack")

# analytical model
from paper_2505_09764_b200 import simulate as fsim  # noqa: E402

t = Topology(2, 4, 900e9, 450e9)
d = workloads.gen_zipf(0, t, 0.8, 10**7)
sched = synth.synthesize_fast(d, t)
fsim.simulate_fast(sched.plan, list(sched.stages), t)
done.append("analytical model")
torch.cuda.synchronize()
print("SANITIZE CASES OK:", "; ".join(done), flush=True)
