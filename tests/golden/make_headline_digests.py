"""Pin the headline config (BASELINE config 5: n = 64 and 128 virtual servers
x 8 GPUs, Zipf 0.8, 2^34 bytes) directly to the REFERENCE.

Runs tiersched (the unmodified reference, imported from /root/reference in
this container) on the benchmark's own seeds and commits SHA-256 digests of

  * the demand matrix (int64 little-endian bytes) -- pins the generator that
    bench.py uses (workloads.zipf_batch_device) to tiersched.gen_zipf;
  * the canonical schedule JSON (tiersched.schedule_to_json, pipeline.py:99)
    -- the whole schedule: moves, reshaped matrix, redistribution tables,
    aux, common_sum and the stripped + sorted stage list;

plus a few plain counts for readable failures.  The JSON at n = 128 is ~100 MB,
so only its digest is committed (tests/golden/headline_digests.json).

    python tests/golden/make_headline_digests.py      # ~1 min at n = 128

The GPU test (tests/test_headline_parity.py) reproduces every digest from the
device output; the CPU suite reproduces them from the C oracle.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "headline_digests.json")

CASES = [(64, 8, s) for s in range(4)] + [(128, 8, s) for s in range(4)]
SKEW, TOTAL = 0.8, 2**34


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    import tiersched as ts

    recs = []
    for n, m, seed in CASES:
        t = ts.Topology(n, m, 900e9, 900e9)
        d = ts.gen_zipf(seed, t, SKEW, TOTAL)
        t0 = time.perf_counter()
        sched = ts.synthesize_fast(d, t)
        el = time.perf_counter() - t0
        js = ts.schedule_to_json(sched)
        recs.append({
            "n": n, "m": m, "seed": seed, "skew": SKEW, "total": TOTAL,
            "demand_sha256": sha(np.ascontiguousarray(d.sizes, dtype="<i8").tobytes()),
            "json_sha256": sha(js.encode()),
            "json_bytes": len(js),
            "n_moves": len(sched.plan.moves),
            "n_raw_stages": len(sched.decomposition.stages),
            "n_stages": len(sched.stages),
            "common_sum": int(sched.decomposition.common_sum),
            "tiersched_seconds": round(el, 2),
        })
        print(recs[-1], flush=True)
    with open(OUT, "w") as fh:
        json.dump({"generator": "tests/golden/make_headline_digests.py (tiersched "
                                "synthesize_fast + schedule_to_json)", "cases": recs}, fh, indent=1)


if __name__ == "__main__":
    main()
