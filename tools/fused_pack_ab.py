"""A/B of the MoE dispatch with and without the fused pack -> send on ONE GPU
(group mode: all ranks of a virtual 2x2 in one cooperative exec launch), so
the row-mapped source reads (cta_copy_rows) are measured against the plain
copy loop on identical traffic, with no NVLink in the way (HBM-local copies
make the per-word index overhead as visible as it can be).

    python tools/fused_pack_ab.py [--tokens 16384] [--row-bytes 8192]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_09764_b200 import Topology  # noqa: E402
from paper_2505_09764_b200.executor import GroupComm, GroupRank  # noqa: E402
from paper_2505_09764_b200.moe import MoEDispatch  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--row-bytes", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--blocks", type=int, default=32)
    args = ap.parse_args()
    T, RB, G = args.tokens, args.row_bytes, 4
    cap = 2 * T * RB * 2
    gen = torch.Generator(device="cuda").manual_seed(1)
    toks = [torch.randint(0, 256, (T, RB), dtype=torch.uint8, device="cuda", generator=gen)
            for _ in range(G)]
    res, outs = {}, {}
    for fused in (False, True):
        group = GroupComm(Topology(2, 2), recv_bytes=cap, staging_bytes=cap, blocks=args.blocks)
        ds = [MoEDispatch(GroupRank(group, s), T, RB, fused_pack=fused) for s in range(G)]

        def step():
            for s, d in enumerate(ds):
                d.route(0)
                if fused:
                    d.rowmap(tokens=toks[s])
                else:
                    d.pack(toks[s])
            Dfull = torch.stack([d.demand_row for d in ds])
            selfb = torch.diagonal(Dfull).clone()
            D = Dfull.clone()
            D.fill_diagonal_(0)
            sends = [t.view(-1) for t in toks] if fused else [d.send for d in ds]
            rows = [(d._tokens, d.row_src, RB) for d in ds] if fused else None
            recvs = group.alltoallv(sends, D, self_bytes=selfb, send_rows=rows)
            for s, d in enumerate(ds):
                d.unpack(D=D, self_sizes=selfb, recv=recvs[s])
            return recvs, Dfull

        for _ in range(3):
            recvs, Dfull = step()
        torch.cuda.synchronize()
        group.check()
        outs[fused] = [recvs[h][: int(Dfull[:, h].sum())].clone() for h in range(G)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        group.check()
        res["fused" if fused else "packed"] = round(e0.elapsed_time(e1) / args.steps, 4)
        group.close()
    same = all(torch.equal(outs[True][h], outs[False][h]) for h in range(G))
    print(json.dumps({"what": "group-mode 2x2 MoE dispatch on one GPU, ms per step (all 4 ranks)",
                      "tokens_per_rank": T, "row_bytes": RB, "ms": res,
                      "expert_inputs_identical": same}))
    if not same:
        raise SystemExit("fused and packed expert inputs differ")


if __name__ == "__main__":
    main()
