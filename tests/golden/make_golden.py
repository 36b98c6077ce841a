"""Generate golden fixtures by running the REFERENCE (tiersched) in this
container.  The fixtures are committed; the GPU box never needs the reference.

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Writes tests/golden/schedules.json.gz (demand-matrix instances with the
reference's canonical schedule JSON), tests/golden/decompositions.json.gz
(server-matrix instances: embedding, raw stages, stripped+sorted stages) and
tests/golden/generators.json.gz (rng / workload generator outputs).
"""

from __future__ import annotations

import argparse
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def _import_ref(path: str):
    sys.dont_write_bytecode = True
    sys.path.insert(0, path)
    import tiersched  # noqa: F401
    from tiersched import rng  # noqa: F401

    return sys.modules["tiersched"]


def _topo(ts, n, m):
    return ts.Topology(n_servers=n, gpus_per_server=m, scaleup_bw=900e9, scaleout_bw=900e9)


HAND6 = [[0, 0, 5, 1, 2, 1], [0, 0, 1, 2, 3, 1], [2, 0, 0, 0, 0, 0],
         [4, 1, 0, 0, 2, 3], [2, 3, 3, 1, 0, 0], [1, 3, 1, 2, 0, 0]]
HAND4 = [[0, 2, 4, 4], [1, 0, 4, 7], [5, 3, 0, 3], [5, 2, 5, 0]]
HAND3 = [[0, 5, 3], [1, 0, 4], [6, 2, 0]]


def demand_instances(ts):
    """(name, n, m, sizes) for the schedule corpus."""
    sys.path.insert(0, REPO)
    from paper_2505_09764_b200.workloads import zipf_sizes

    out = [("hand6", 3, 2, np.array(HAND6, np.int64)),
           ("hand4_m1", 4, 1, np.array(HAND4, np.int64)),
           ("hand3_m1", 3, 1, np.array(HAND3, np.int64)),
           ("kat_2x1", 2, 1, np.array([[0, 40], [60, 0]], np.int64)),
           ("zeros_2x2", 2, 2, np.zeros((4, 4), np.int64)),
           ("single_2x3", 2, 3, np.eye(6, k=4, dtype=np.int64) * 17)]
    for n, m in [(2, 2), (3, 2), (4, 3), (3, 4)]:
        out.append((f"adversarial_{n}x{m}", n, m, ts.gen_adversarial(_topo(ts, n, m), 77).sizes))
    # c8-style corpus (test_acceptance.py:278-295)
    for seed in range(300):
        n, m = 2 + seed % 4, 1 + seed % 3
        out.append((f"c8_{seed}", n, m, ts.gen_uniform(seed, _topo(ts, n, m), 1000).sizes))
    # BASELINE configs 1/2/4 shapes: uniform (zipf skew 0) and skewed, 2x4 / 4x2
    for n, m in [(2, 4), (4, 2), (2, 2), (2, 1)]:
        t = _topo(ts, n, m)
        for seed in range(4):
            out.append((f"uniform64M_{n}x{m}_{seed}", n, m,
                        ts.gen_zipf(seed, t, 0.0, 67_108_864).sizes))
            out.append((f"zipf08_{n}x{m}_{seed}", n, m, ts.gen_zipf(seed, t, 0.8, 1 << 30).sizes))
            # alpha = 1.2 needs the restated generator (reference rejects >= 1)
            out.append((f"zipf12_256M_{n}x{m}_{seed}", n, m,
                        zipf_sizes(seed, n * m, 1.2, 268_435_456)))
            out.append((f"random_{n}x{m}_{seed}", n, m, ts.gen_uniform(seed, t, 1_198_372).sizes))
    # larger m (wide tiles) and huge values near the 2^62 guard
    for seed in range(6):
        out.append((f"wide_2x16_{seed}", 2, 16,
                    ts.gen_zipf(seed, _topo(ts, 2, 16), 0.9, 10**12 + seed).sizes))
        out.append((f"big_3x3_{seed}", 3, 3,
                    ts.gen_zipf(seed, _topo(ts, 3, 3), 0.5, (1 << 61) + seed).sizes))
    # config-5 shapes (Zipf 0.8, 2^34 total)
    for n, seeds in [(16, 3), (32, 1)]:
        for seed in range(seeds):
            out.append((f"cfg5_{n}x8_{seed}", n, 8,
                        ts.gen_zipf(seed, _topo(ts, n, 8), 0.8, 2**34).sizes))
    return out


def server_instances(ts):
    from tiersched import rng

    out = []
    for seed in range(300):  # c1-style corpus (test_acceptance.py:44-50)
        n = 2 + seed % 15
        draws = rng.stream(seed, n * n) % np.uint64(997)
        s = draws.astype(np.int64).reshape(n, n)
        np.fill_diagonal(s, 0)
        out.append((f"c1_{seed}", s))
    out.append(("hand4", np.array(HAND4, np.int64)))
    out.append(("hand3", np.array(HAND3, np.int64)))
    out.append(("diag_aux", np.array([[0, 0, 0], [0, 0, 5], [0, 5, 0]], np.int64)))
    out.append(("zeros4", np.zeros((4, 4), np.int64)))
    for seed, n in enumerate((24, 40)):  # a few larger server matrices
        draws = rng.stream(1000 + seed, n * n) % np.uint64(1 << 40)
        s = draws.astype(np.int64).reshape(n, n)
        np.fill_diagonal(s, 0)
        out.append((f"large_{n}", s))
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    ts = _import_ref(args.ref)

    recs = []
    for name, n, m, sizes in demand_instances(ts):
        d = ts.DemandMatrix(n_servers=n, gpus_per_server=m, sizes=np.asarray(sizes, np.int64))
        sched = ts.synthesize_fast(d, _topo(ts, n, m))
        recs.append({"name": name, "n": n, "m": m, "D": d.sizes.tolist(),
                     "json": ts.schedule_to_json(sched)})
    with gzip.open(os.path.join(HERE, "schedules.json.gz"), "wt") as fh:
        json.dump(recs, fh)

    drecs = []
    for name, s in server_instances(ts):
        sm = ts.ServerMatrix(totals=s)
        emb, aux = ts.embed_doubly_stochastic(sm)
        dec = ts.decompose_server_matrix(sm)
        stripped = ts.sort_stages_ascending(ts.strip_auxiliary(list(dec.stages), dec.aux))
        st = lambda sts: [[int(x.weight), [list(map(int, e)) for e in x.edges]] for x in sts]  # noqa: E731
        drecs.append({"name": name, "S": s.tolist(), "embedded": emb.tolist(),
                      "aux": aux.tolist(), "common_sum": int(dec.common_sum),
                      "raw": st(dec.stages), "sorted": st(stripped)})
    with gzip.open(os.path.join(HERE, "decompositions.json.gz"), "wt") as fh:
        json.dump(drecs, fh)

    from tiersched import rng

    t42 = _topo(ts, 4, 2)
    gens = {
        "stream0_first": int(rng.stream(0, 1)[0]),
        "stream_7_16_off3": [int(x) for x in rng.stream(7, 16, 3)],
        "uniform_5_4x2_100": ts.gen_uniform(5, t42, 100).sizes.tolist(),
        "zipf": [{"seed": s, "skew": k, "total": tot, "n": 4, "m": 2,
                  "sizes": ts.gen_zipf(s, t42, k, tot).sizes.tolist()}
                 for s, k, tot in [(3, 0.9, 10_000_000_001), (1, 0.0, 10_007), (2, 0.5, 12345),
                                   (0, 0.8, 1 << 30), (9, 0.99, 999)]],
    }
    with gzip.open(os.path.join(HERE, "generators.json.gz"), "wt") as fh:
        json.dump(gens, fh)
    print(f"{len(recs)} schedules, {len(drecs)} decompositions written to {HERE}")


if __name__ == "__main__":
    main()
