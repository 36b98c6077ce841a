"""GPU synthesis parity: the sm_100a kernels vs the reference and the oracle.

* every golden schedule (made by tiersched) -> identical canonical JSON;
* every golden server-matrix decomposition -> identical aux / raw / sorted;
* config-5 shapes (n = 16..128, m = 8) and random batches -> packed arrays
  identical to the C oracle's (bit-exact, all int64);
* validation errors map to ValidationError / status 2.
"""

from __future__ import annotations

from collections import defaultdict

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2505_09764_b200 import (DemandMatrix, ServerMatrix, Topology, ValidationError,
                                   schedule_to_json, workloads)
from paper_2505_09764_b200 import synth

pytestmark = pytest.mark.gpu


def _packed_equal(gpu_bufs: synth.SynthBuffers, ref: dict, B: int, n: int, m: int,
                  only=None):
    """Compare device output with the oracle's, matrix by matrix."""
    h = {k: getattr(gpu_bufs, k).cpu().numpy() for k in (
        "balanced", "server", "move_count", "common_sum", "aux", "n_raw", "n_stages",
        "status", "stage_weight", "stage_perm", "stage_bytes", "stage_order")}
    moves = gpu_bufs.moves.cpu().numpy().view(oracle.MOVE_DTYPE).reshape(ref["moves"].shape)
    for b in (range(B) if only is None else only):
        assert h["status"][b] == ref["status"][b] == 0, b
        for k in ("balanced", "server", "move_count", "aux"):
            assert np.array_equal(h[k][b], ref[k][b]), (k, b)
        cnt = ref["move_count"][b]
        for t in np.flatnonzero(cnt):
            assert np.array_equal(moves[b, t, :cnt[t]], ref["moves"][b, t, :cnt[t]]), (b, t)
        assert h["common_sum"][b] == ref["common_sum"][b]
        k = int(ref["n_raw"][b])
        s = int(ref["n_stages"][b])
        assert h["n_raw"][b] == k and h["n_stages"][b] == s, b
        assert np.array_equal(h["stage_weight"][b, :k], ref["stage_weight"][b, :k]), b
        assert np.array_equal(h["stage_perm"][b, :k], ref["stage_perm"][b, :k]), b
        assert np.array_equal(h["stage_bytes"][b, :k], ref["stage_bytes"][b, :k]), b
        assert np.array_equal(h["stage_order"][b, :s], ref["stage_order"][b, :s]), b


def test_gpu_matches_every_golden_schedule(golden_schedules):
    groups = defaultdict(list)
    for rec in golden_schedules:
        groups[(rec["n"], rec["m"])].append(rec)
    total = 0
    for (n, m), recs in groups.items():
        D = torch.tensor(np.array([r["D"] for r in recs], dtype=np.int64), device="cuda")
        packed = synth.synthesize_packed(D, n, m).host()
        for rec, p in zip(recs, packed):
            assert p.status == 0, rec["name"]
            assert schedule_to_json(p.to_schedule()) == rec["json"], rec["name"]
            total += 1
    assert total == len(golden_schedules)


def test_gpu_matches_every_golden_decomposition(golden_decompositions):
    for rec in golden_decompositions:
        s = ServerMatrix(np.array(rec["S"], dtype=np.int64))
        dec = synth.decompose_server_matrix(s)
        assert dec.common_sum == rec["common_sum"], rec["name"]
        assert dec.aux.tolist() == rec["aux"], rec["name"]
        raw = [[st.weight, [list(e) for e in st.edges]] for st in dec.stages]
        assert raw == rec["raw"], rec["name"]
        emb, aux = synth.embed_doubly_stochastic(s)
        assert emb.tolist() == rec["embedded"], rec["name"]
        again = synth.decompose(emb)
        assert [[st.weight, [list(e) for e in st.edges]] for st in again] == rec["raw"]


@pytest.mark.parametrize("n,B", [(16, 64), (32, 16), (64, 4), (128, 2), (64, 40), (128, 17),
                                 (128, 24), (80, 30), (100, 41), (128, 40)])
def test_gpu_matches_oracle_config5_shapes(n, B):
    m = 8
    G = n * m
    D = np.stack([workloads.zipf_sizes(100 + b, G, 0.8, 2**34) for b in range(B)])
    ref = oracle.synthesize_batch(D, n, m)
    bufs = synth.synthesize_packed(torch.from_numpy(D).cuda(), n, m)
    _packed_equal(bufs, ref, B, n, m)


@pytest.mark.parametrize("n,m", [(2, 4), (4, 2), (2, 1), (2, 2), (3, 5), (5, 3), (8, 8), (2, 16),
                                 (3, 32), (2, 64), (7, 6)])
def test_gpu_matches_oracle_random_batches(n, m):
    rng = np.random.default_rng(n * 100 + m)
    B = 257
    G = n * m
    D = rng.integers(0, 1000, size=(B, G, G), dtype=np.int64)
    D[rng.random(D.shape) < 0.5] = 0  # sparse: empty stages, aux on the diagonal
    D[B // 2:] = rng.integers(0, 1 << 40, size=(B - B // 2, G, G))
    D[:, np.arange(G), np.arange(G)] = 0
    ref = oracle.synthesize_batch(D, n, m)
    bufs = synth.synthesize_packed(torch.from_numpy(D).cuda(), n, m)
    _packed_equal(bufs, ref, B, n, m)


def test_gpu_api_synthesize_fast_and_balance_plan(golden_schedules):
    rec = next(r for r in golden_schedules if r["name"] == "hand6")
    d = DemandMatrix(3, 2, np.array(rec["D"], np.int64))
    t = Topology(3, 2)
    assert schedule_to_json(synth.synthesize_fast(d, t)) == rec["json"]
    plan = synth.build_balance_plan(d, t)
    full = synth.synthesize_fast(d, t).plan
    assert plan.moves == full.moves
    assert np.array_equal(plan.reshaped.sizes, full.reshaped.sizes)
    batch = synth.synthesize_fast_batch([d, d], t)
    assert schedule_to_json(batch[1]) == rec["json"]


def test_gpu_validation_errors_and_status():
    n, m = 2, 2
    D = np.zeros((4, 4, 4), np.int64)
    D[0, 0, 1] = 5
    D[1, 2, 2] = 3          # diagonal
    D[2, 0, 3] = -1         # negative
    D[3, 0, 2] = 1 << 61    # total >= 2^62
    D[3, 1, 3] = 1 << 61
    bufs = synth.synthesize_packed(torch.from_numpy(D).cuda(), n, m)
    assert bufs.status.cpu().tolist() == [0, 2, 2, 2]
    with pytest.raises(ValidationError):
        synth.decompose(np.array([[1, 2], [0, 1]], np.int64))


@pytest.mark.parametrize("m", [4, 8, 16])
def test_gpu_balance_wide_cells_and_invalid_tiles(m):
    """The register-staged balance kernel's exact fallback: tiles with cells
    at or above 2^(62 - ceil(log2 m^2)) (valid, and past the 2^62 guard), negative
    cells and non-zero diagonals, next to ordinary tiles of the same CTA."""
    n, B = 3, 12
    G = n * m
    rng = np.random.default_rng(m)
    D = rng.integers(0, 1 << 30, size=(B, G, G), dtype=np.int64)
    D[:, np.arange(G), np.arange(G)] = 0
    big = 1 << (62 - int(np.ceil(np.log2(m * m))))  # first width past the fast path
    D[1, 0, m + 1] = big                     # wide cell, total stays below 2^62
    D[2, 1, 2 * m] = (1 << 61) - 5           # wide cells over 2^62 in one tile
    D[2, 2, 2 * m + 1] = (1 << 61) - 3
    D[3, 0, 1] = 7                           # diagonal tile entry (0, 1) is off-diagonal: valid
    D[4, m + 2, m + 2] = 9                   # diagonal cell
    D[5, 2, m + 3] = -1                      # negative
    D[6, 2 * m + 1, 1] = big - 1
    ref = oracle.synthesize_batch(D, n, m)
    bufs = synth.synthesize_packed(torch.from_numpy(D).cuda(), n, m)
    st = bufs.status.cpu().tolist()
    assert st == ref["status"].tolist()
    _packed_equal(bufs, ref, B, n, m, only=[b for b in range(B) if st[b] == 0])
    assert st[2] == 2 and st[4] == 2 and st[5] == 2 and st[1] == 0 and st[6] == 0


def test_gpu_misaligned_demand_view_is_rejected():
    """Even m moves 16-byte pairs: an 8-byte-offset view of D is refused with
    ValidationError (never a device fault), and the aligned copy works."""
    n, m, B = 3, 2, 2
    G = n * m
    base = torch.zeros(B * G * G + 1, dtype=torch.int64, device="cuda")
    D = base[1:].view(B, G, G)
    D[:, 0, 3] = 5
    assert D.data_ptr() % 16 == 8
    with pytest.raises(ValidationError):
        synth.synthesize_packed(D, n, m)
    bufs = synth.synthesize_packed(D.clone(), n, m)
    assert bufs.status.cpu().tolist() == [0, 0]


def test_gpu_deterministic_across_runs():
    n, m, B = 32, 8, 8
    D = np.stack([workloads.zipf_sizes(b, n * m, 1.2, 2**34) for b in range(B)])
    Dt = torch.from_numpy(D).cuda()
    a = synth.synthesize_packed(Dt, n, m).host()
    b = synth.synthesize_packed(Dt, n, m).host()
    for pa, pb in zip(a, b):
        assert pa.n_raw == pb.n_raw and pa.n_stages == pb.n_stages
        for k in ("stage_weight", "stage_perm", "stage_bytes", "stage_order", "balanced"):
            assert np.array_equal(getattr(pa, k), getattr(pb, k)), k


def test_gpu_compact_layout_matches_golden(golden_schedules):
    """The batch product layout (no per-edge stage bytes: the aux run-out
    table; balanced tiles as changed-cell masks + values) decodes to the
    reference's canonical JSON, on device and through the pinned-host path."""
    groups = defaultdict(list)
    for rec in golden_schedules:
        if rec["m"] <= 8:
            groups[(rec["n"], rec["m"])].append(rec)
    total = 0
    for (n, m), recs in groups.items():
        Dn = np.array([r["D"] for r in recs], dtype=np.int64)
        D = torch.tensor(Dn, device="cuda")
        bufs = synth.SynthBuffers(len(recs), n, m, D.device, stage_bytes=False, compact=True)
        packed = synth.synthesize_packed(D, n, m, bufs).host()
        hs = synth.synthesize_host_batch(torch.from_numpy(Dn).pin_memory(), n, m, chunk=7)
        for b, (rec, p) in enumerate(zip(recs, packed)):
            assert p.status == 0, rec["name"]
            assert schedule_to_json(p.to_schedule()) == rec["json"], rec["name"]
            assert schedule_to_json(hs.packed(b, Dn[b]).to_schedule()) == rec["json"], rec["name"]
            total += 1
    assert total > 300


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_gpu_host_pipeline_stream_matches_oracle(depth):
    """HostSynthPipeline.run: a stream of distinct batches with `depth`
    buffer sets in rotation (several batches in flight) -- every batch's
    compact host result equals the oracle's."""
    n, m, B, K = 12, 4, 9, 5
    G = n * m
    Ds = []
    for t in range(K):
        rng = np.random.default_rng(100 + t)
        D = rng.integers(0, 1 << 32, size=(B, G, G), dtype=np.int64)
        D[rng.random(D.shape) < 0.2] = 0
        D[:, np.arange(G), np.arange(G)] = 0
        Ds.append(D)
    pipe = synth.HostSynthPipeline(B, n, m, chunk=4, depth=depth)
    outs = [synth.HostSchedules(B, n, m) for _ in range(max(2, depth))]
    done = pipe.run([torch.from_numpy(D).pin_memory() for D in Ds],
                    [outs[t % len(outs)] for t in range(K)])
    assert len(done) == K
    # each result is read before its HostSchedules object is reused: check the
    # last len(outs) batches (the earlier ones were overwritten by design)
    for t in range(K - len(outs), K):
        hs, D = done[t], Ds[t]
        ref = oracle.synthesize_batch(D, n, m)
        for b in range(B):
            p = hs.packed(b, D[b])
            want = oracle.packed_fields(ref, b, n, m)
            for key in ("balanced", "move_count", "stage_weight", "stage_perm", "stage_bytes",
                        "stage_order"):
                assert np.array_equal(getattr(p, key), want[key]), (key, t, b)
            used = np.arange(want["moves"].shape[1])[None, :] < want["move_count"][:, None]
            assert np.array_equal(p.moves[used], want["moves"][used]), (t, b)


@pytest.mark.parametrize("n,m", [(16, 8), (8, 8), (5, 3), (3, 1), (3, 16), (2, 12)])
def test_gpu_compact_layout_matches_oracle(n, m):
    rng = np.random.default_rng(7 * n + m)
    B, G = 33, n * m
    D = rng.integers(0, 1 << 30, size=(B, G, G), dtype=np.int64)
    D[rng.random(D.shape) < 0.3] = 0
    D[:, np.arange(G), np.arange(G)] = 0
    ref = oracle.synthesize_batch(D, n, m)
    hs = synth.synthesize_host_batch(torch.from_numpy(D).pin_memory(), n, m, chunk=10)
    if m <= 8:  # m > 8 ships the balanced matrix itself (no 64-bit tile masks)
        assert hs.nbytes() < synth.SynthBuffers(B, n, m, torch.device("cuda")).output_nbytes()
    for b in range(B):
        p = hs.packed(b, D[b])
        want = oracle.packed_fields(ref, b, n, m)
        for key in ("balanced", "server", "move_count", "aux", "stage_weight", "stage_perm",
                    "stage_bytes", "stage_order"):
            assert np.array_equal(getattr(p, key), want[key]), (key, b)
        assert (p.status, p.common_sum, p.n_raw, p.n_stages) == (
            want["status"], want["common_sum"], want["n_raw"], want["n_stages"]), b
