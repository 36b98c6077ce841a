"""Generate the simulator golden fixtures by running the REFERENCE
(tiersched) in this container.  The fixture is committed; the GPU box never
needs the reference.

    python tests/golden/make_sim_golden.py [--ref /root/reference/pkg/src]

Writes tests/golden/simulate.json.gz: demand-matrix instances over assorted
topologies (bandwidth ratios, wakeup delays) with the reference's
    simulate_fast(plan, stages, t)            (simulate.py:107-193)
    simulate_spreadout(s, t) / (s, t, d)      (simulate.py:196-242)
    optimal_time / fast_worstcase_time / ratio_bound /
    intra_assumption_holds                    (bounds.py:42-87)
    spreadout_stages weights                  (spreadout.py:19-31)
Floats are stored as float.hex() so parity is checked bit for bit.
"""

from __future__ import annotations

import argparse
import gzip
import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def _import_ref(path: str):
    sys.dont_write_bytecode = True
    sys.path.insert(0, path)
    import tiersched  # noqa: F401

    return sys.modules["tiersched"]


# (n, m, scaleup_bw, scaleout_bw, wakeup_delay)
TOPOS = [
    (2, 1, 100.0, 10.0, 0.5), (2, 2, 900e9, 900e9, 0.0), (2, 4, 900e9, 900e9, 0.0),
    (4, 2, 900e9, 900e9, 2e-6), (3, 2, 450e9, 50e9, 0.0), (3, 4, 400e9, 50e9, 1e-5),
    (4, 8, 450e9, 50e9, 0.0), (5, 4, 800e9, 50e9, 3e-6), (5, 3, 250e9, 50e9, 0.0),
    (8, 1, 900e9, 100e9, 1e-6), (6, 2, 3e11, 1e11, 0.0), (16, 8, 900e9, 400e9, 5e-6),
    (7, 5, 1e12, 2.5e11, 0.0), (3, 8, 123456789.0, 98765432.1, 0.125),
]


def instances(ts):
    sys.path.insert(0, REPO)
    from paper_2505_09764_b200.workloads import zipf_sizes

    out = []
    for ti, (n, m, b1, b2, a) in enumerate(TOPOS):
        t = ts.Topology(n, m, scaleup_bw=b1, scaleout_bw=b2, wakeup_delay=a)
        G = n * m
        cases = [("zipf0.8", ts.gen_zipf(ti, t, 0.8, 10_000_000_000).sizes),
                 ("uniform", ts.gen_uniform(ti + 1, t, 5_000_000).sizes),
                 ("adversarial", ts.gen_adversarial(t, 1_000_003 + ti).sizes),
                 ("zipf1.2", zipf_sizes(ti + 7, G, 1.2, 268_435_456))]
        rs = np.random.default_rng(ti)
        sp = rs.integers(0, 1 << 20, (G, G)).astype(np.int64)
        sp[rs.random((G, G)) < 0.7] = 0
        np.fill_diagonal(sp, 0)
        cases.append(("sparse", sp))
        if G <= 16:
            # products cell * r >= 2^63: split_deliveries' exact-integer path
            huge = rs.integers(1 << 51, 1 << 53, (G, G)).astype(np.int64)
            np.fill_diagonal(huge, 0)
            cases.append(("huge", huge))
        intra = np.zeros((G, G), np.int64)
        for i in range(n):
            blk = rs.integers(0, 10**9, (m, m))
            intra[i * m:(i + 1) * m, i * m:(i + 1) * m] = blk
        np.fill_diagonal(intra, 0)
        cases.append(("intra_only", intra))
        cases.append(("zeros", np.zeros((G, G), np.int64)))
        for name, sizes in cases:
            out.append((f"{name}_{n}x{m}_t{ti}", n, m, (b1, b2, a), np.asarray(sizes, np.int64)))
    # the hand-checked pipeline KAT (test_simulate.py:105-122)
    out.append(("kat_2x1", 2, 1, (100.0, 10.0, 0.5), np.array([[0, 40], [60, 0]], np.int64)))
    return out


def _hex(xs):
    return [float(x).hex() for x in xs]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    ts = _import_ref(args.ref)
    rows = []
    for name, n, m, (b1, b2, a), sizes in instances(ts):
        t = ts.Topology(n, m, scaleup_bw=b1, scaleout_bw=b2, wakeup_delay=a)
        d = ts.DemandMatrix(n, m, sizes)
        sched = ts.synthesize_fast(d, t)
        line = ts.simulate_fast(sched.plan, list(sched.stages), t)
        server = ts.reduce_to_server_level(d, t)
        so = ts.simulate_spreadout(server, t)
        so_d = ts.simulate_spreadout(server, t, demand=d)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            t_opt = ts.optimal_time(server, t)
            t_worst = ts.fast_worstcase_time(server, t)
        rows.append({
            "name": name, "n": n, "m": m, "topo": _hex((b1, b2, a)),
            "sizes": sizes.tolist(),
            "fast": {"t_balance": float(line.t_balance).hex(),
                     "t_intra_a2a": float(line.t_intra_a2a).hex(),
                     "scale_out": _hex(line.scale_out),
                     "redistribution": _hex(line.redistribution),
                     "total": float(line.total).hex()},
            "spreadout": {"scale_out": _hex(so.scale_out), "total": float(so.total).hex()},
            "spreadout_demand": {"scale_out": _hex(so_d.scale_out),
                                 "total": float(so_d.total).hex()},
            "spreadout_weights": [int(st.weight) for st in ts.spreadout_stages(server)],
            "spreadout_units": int(ts.spreadout_completion_units(server)),
            "t_optimal": float(t_opt).hex(), "t_worstcase": float(t_worst).hex(),
            "ratio_bound": float(ts.ratio_bound(t)).hex(),
            "assumption_ok": bool(ts.intra_assumption_holds(server)),
        })
    path = os.path.join(HERE, "simulate.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(rows, f, separators=(",", ":"))
    print(f"{len(rows)} instances -> {path}")


if __name__ == "__main__":
    main()
