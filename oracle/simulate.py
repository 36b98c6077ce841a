"""CPU ORACLE for the analytical cost model -- test infrastructure only.

Restates, over the packed schedule form (oracle.packed_fields), the
reference's
  * simulate_fast        /root/reference/pkg/src/tiersched/simulate.py:107-193
    - step_cost          simulate.py:58-66
    - intra_phase_time   simulate.py:69-90 (per (server, gpu) send/recv sums)
    - _intra_alltoall_time simulate.py:93-104
    - split_deliveries   balance.py:177-207 (floor(cell*r/T), last gets the rest)
  * simulate_spreadout   simulate.py:196-242
  * spreadout_stages     spreadout.py:19-31 (weights only)
  * optimal_time / fast_worstcase_time / ratio_bound / intra_assumption_holds
                         bounds.py:27-87
in plain Python integers and floats with the reference's operation order,
so results are bit-identical.  Pinned against tests/golden/simulate.json.gz
(generated from the reference itself by tests/golden/make_sim_golden.py).
"""

from __future__ import annotations

import numpy as np


def step_cost(nbytes, bw: float, wake: float) -> float:
    if nbytes == 0:
        return 0.0
    return wake + nbytes / bw


def _present(sb: int) -> bool:
    return sb != 0  # packed form: 0 = no edge, -1 = a zero-byte edge


def simulate_fast(p: dict, b1: float, b2: float, wake: float) -> dict:
    """p: oracle.packed_fields(...) of one matrix.  Returns the Timeline
    fields, or {"error": "validation"|"invariant"}."""
    n, m = p["n"], p["m"]
    G = n * m
    bal = np.asarray(p["balanced"], dtype=np.int64)
    order = [int(x) for x in p["stage_order"]]
    weights = [int(p["stage_weight"][k]) for k in order]
    if any(a > b for a, b in zip(weights, weights[1:])):
        return {"error": "validation"}
    # balance moves: per (server, gpu) send / receive totals
    send: dict = {}
    recv: dict = {}
    slots = p["moves"].shape[1] if p["moves"].ndim == 2 else 1
    t = 0
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            for s in range(int(p["move_count"][t])):
                mv = p["moves"][t][s] if slots else None
                f, to, x = int(mv["from_gpu"]), int(mv["to_gpu"]), int(mv["bytes"])
                send[(i, f)] = send.get((i, f), 0) + x
                recv[(i, to)] = recv.get((i, to), 0) + x
            t += 1
    worst = 0
    for table in (send, recv):
        for v in table.values():
            worst = max(worst, v)
    t_balance = step_cost(worst, b1, wake)
    worst = 0
    for i in range(n):
        blk = bal[i * m:(i + 1) * m, i * m:(i + 1) * m]
        if blk.any():
            worst = max(worst, int(blk.sum(axis=1).max()), int(blk.sum(axis=0).max()))
    t_intra = step_cost(worst, b1, wake)
    # per-pair deliveries in stage order
    pair: dict = {}
    for k, raw in enumerate(order):
        for i in range(n):
            sb = int(p["stage_bytes"][raw][i])
            if _present(sb):
                j = int(p["stage_perm"][raw][i])
                pair.setdefault((i, j), []).append((k, max(sb, 0)))
    for (i, j), ent in pair.items():
        if i == j or j >= n:
            return {"error": "invariant"}
        tab = bal[i * m:(i + 1) * m, j * m:(j + 1) * m]
        if sum(b for _, b in ent) != int(tab.sum()):
            return {"error": "invariant"}
    for i in range(n):
        for j in range(n):
            if i != j and bal[i * m:(i + 1) * m, j * m:(j + 1) * m].sum() > 0 and (i, j) not in pair:
                return {"error": "invariant"}
    S = len(order)
    out = []
    for raw in order:
        mx = 0
        for i in range(n):
            sb = int(p["stage_bytes"][raw][i])
            if _present(sb):
                mx = max(mx, max(sb, 0))
        out.append(step_cost(mx / m, b2, wake))
    rw = [0] * S
    for (i, j), ent in pair.items():
        tab = [[int(x) for x in row] for row in bal[i * m:(i + 1) * m, j * m:(j + 1) * m]]
        T = sum(map(sum, tab))
        if T == 0:
            continue
        acc = [[0] * m for _ in range(m)]
        for e, (k, r) in enumerate(ent):
            last = e == len(ent) - 1
            piece = [[(tab[a][c] - acc[a][c]) if last else tab[a][c] * r // T for c in range(m)]
                     for a in range(m)]
            for a in range(m):
                for c in range(m):
                    acc[a][c] += piece[a][c]
            for a in range(m):
                piece[a][a] = 0
            if any(any(row) for row in piece):
                w = max(max(sum(row) for row in piece),
                        max(sum(piece[a][c] for a in range(m)) for c in range(m)))
                rw[k] = max(rw[k], w)
    redist = [step_cost(w, b1, wake) for w in rw]
    if not S:
        return {"t_balance": t_balance, "t_intra_a2a": t_intra, "scale_out": [],
                "redistribution": [], "total": t_balance + t_intra}
    total = t_balance + max(out[0], t_intra)
    for k in range(1, S):
        total += max(out[k], redist[k - 1])
    total += redist[-1]
    floor = int(p["common_sum"]) / (m * b2)
    if total < floor * (1 - 1e-12):
        return {"error": "invariant"}
    return {"t_balance": t_balance, "t_intra_a2a": t_intra, "scale_out": out,
            "redistribution": redist, "total": total}


def _off(server: np.ndarray) -> list[list[int]]:
    n = server.shape[0]
    return [[0 if a == b else int(server[a][b]) for b in range(n)] for a in range(n)]


def simulate_spreadout(server: np.ndarray, m: int, b2: float, wake: float,
                       demand: np.ndarray | None = None) -> dict:
    n = server.shape[0]
    off = _off(server)
    dur = []
    for shift in range(1, n):
        if demand is None:
            gov = max(off[s][(s + shift) % n] for s in range(n)) / m
        else:
            gov = 0
            for s in range(n):
                d = (s + shift) % n
                blk = demand[s * m:(s + 1) * m, d * m:(d + 1) * m]
                if blk.any():
                    gov = max(gov, int(blk.sum(axis=1).max()), int(blk.sum(axis=0).max()))
        dur.append(step_cost(gov, b2, wake))
    # Python >= 3.12 sum() of floats is Neumaier-compensated (the reference's
    # own interpreter); the device kernel restates that algorithm
    return {"scale_out": dur, "total": sum(dur)}


def spreadout_weights(server: np.ndarray) -> list[int]:
    n = server.shape[0]
    off = _off(server)
    return [max(off[s][(s + shift) % n] for s in range(n)) for shift in range(1, n)]


def bounds(server: np.ndarray, m: int, b1: float, b2: float) -> dict:
    n = server.shape[0]
    off = _off(server)
    rows = [sum(r) for r in off]
    cols = [sum(off[a][b] for a in range(n)) for b in range(n)]
    mrc = max(max(rows), max(cols))
    row_max = max(rows)
    t0 = (m - 1) * row_max / (m * b1)
    t1 = row_max / (n * b1)
    t2 = mrc / (m * b2)
    t3 = max(max(r) for r in off) / (m * b1)
    ok = all(n * int(server[i][i]) <= rows[i] for i in range(n))
    return {"t_optimal": mrc / (m * b2), "t_worstcase": t0 + t1 + t2 + t3,
            "ratio_bound": 1.0 + (b2 / b1) * (m + m / n), "assumption_ok": ok}
