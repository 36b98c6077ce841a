"""Stage-level building blocks and IO helpers of the drop-in API.

GPU: find_perfect_matching / balance_senders / strip_auxiliary /
sort_stages_ascending (device kernels, csrc/stages.cu + the balance kernel)
against the reference's own outputs (tests/golden/blocks.json.gz, made by
tests/golden/make_blocks_golden.py).  CPU: save_matrix / load_matrix /
load_trace round trips and their ValidationError cases (model.py:194-255),
merge_peer, and that every name the reference exports resolves.
"""

from __future__ import annotations

import gzip
import json
import os

import numpy as np
import pytest

from conftest import REPO

GOLDEN = os.path.join(REPO, "tests", "golden", "blocks.json.gz")


def _golden():
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)


def _as_stages(items):
    from paper_2505_09764_b200 import PermutationStage

    return [PermutationStage(weight=it["weight"], edges=tuple(tuple(e) for e in it["edges"]))
            for it in items]


def _plain(stages):
    return [{"weight": int(s.weight), "edges": [[int(a), int(b), int(c)] for a, b, c in s.edges]}
            for s in stages]


def test_reference_names_all_resolve():
    import paper_2505_09764_b200 as fb

    # tiersched.__all__ (/root/reference/pkg/src/tiersched/__init__.py:76-129)
    names = ["BalancePlan", "BoundsReport", "Decomposition", "DemandMatrix",
             "InternalInvariantError", "IntraMove", "PermutationStage", "Schedule", "ServerMatrix",
             "SpreadoutSchedule", "TileView", "Timeline", "Topology", "ValidationError",
             "algorithmic_bandwidth", "balance_senders", "bounds_report", "build_balance_plan",
             "decompose", "decompose_server_matrix", "embed_doubly_stochastic",
             "fast_worstcase_time", "find_perfect_matching", "gen_adversarial", "gen_uniform",
             "gen_zipf", "intra_assumption_holds", "intra_phase_time", "load_matrix", "load_trace",
             "max_rc", "merge_peer", "optimal_time", "ratio_bound", "reduce_to_server_level",
             "save_matrix", "schedule_from_json", "schedule_to_json", "simulate_fast",
             "simulate_spreadout", "sort_stages_ascending", "split_deliveries",
             "spreadout_completion_units", "spreadout_intra", "spreadout_stages",
             "stage_redistribution", "step_cost", "strip_auxiliary", "synthesize_fast",
             "synthesize_spreadout", "tile", "validate_topology"]
    missing = [n for n in names if n not in fb.__all__]
    assert not missing, missing


def test_matrix_io_round_trip(tmp_path):
    import paper_2505_09764_b200 as fb

    d = fb.gen_uniform(3, fb.Topology(2, 3), 12345)
    for name in ("m.json", "m.csv", "trace.txt"):
        p = str(tmp_path / name)
        fb.save_matrix(d, p)
        back = fb.load_matrix(p)
        assert (back.n_servers, back.gpus_per_server) == (2, 3)
        assert np.array_equal(back.sizes, d.sizes)
        assert np.array_equal(fb.load_trace(p).sizes, d.sizes)
    with open(tmp_path / "m.json") as f:  # canonical: sorted keys, no spaces
        assert f.read().startswith('{"m":3,"n":2,"sizes":[[')


def test_matrix_io_errors(tmp_path):
    import paper_2505_09764_b200 as fb

    cases = {"missing.json": None, "bad.json": "{not json", "keys.json": '{"n": 2}',
             "nohdr.csv": "1,2\n3,4\n", "badhdr.csv": "# n=x m=1\n0,1\n1,0\n",
             "body.csv": "# n=2 m=1\n0,a\n1,0\n", "ragged.csv": "# n=2 m=1\n0,1\n1\n",
             "diag.csv": "# n=2 m=1\n5,1\n1,0\n"}
    for name, text in cases.items():
        p = tmp_path / name
        if text is not None:
            p.write_text(text)
        with pytest.raises(fb.ValidationError):
            fb.load_matrix(str(p))


def test_merge_peer():
    from paper_2505_09764_b200.synth import merge_peer
    from paper_2505_09764_b200 import ValidationError

    t = np.array([[3, 1], [2, 1]], np.int64)
    scalar, red = merge_peer(t)
    assert np.array_equal(scalar, np.diag([4, 3])) and np.array_equal(red, t)
    with pytest.raises(ValidationError):
        merge_peer(np.array([[5, 0], [1, 0]], np.int64))


@pytest.mark.gpu
def test_find_perfect_matching_matches_reference():
    import paper_2505_09764_b200 as fb

    g = _golden()["matching"]
    assert sum(c["match"] == "error" for c in g) >= 2
    for c in g:
        sp = np.array(c["support"], dtype=bool)
        if c["match"] == "error":
            with pytest.raises(fb.InternalInvariantError):
                fb.find_perfect_matching(sp)
            continue
        r = fb.find_perfect_matching(sp)
        assert [r[u] for u in range(sp.shape[0])] == c["match"]
    # full 4x4 support -> anti-diagonal pins the DFS order (test_birkhoff.py:92-98)
    assert fb.find_perfect_matching(np.ones((4, 4), bool)) == {0: 3, 1: 2, 2: 1, 3: 0}


@pytest.mark.gpu
def test_balance_senders_matches_reference():
    import paper_2505_09764_b200 as fb

    for c in _golden()["balance"]:
        e = np.array(c["tile"], np.int64)
        bal, moves = fb.balance_senders(fb.TileView(src_server=1, dst_server=0, entries=e))
        assert np.array_equal(bal, np.array(c["balanced"], np.int64))
        got = [[mv.server, mv.from_gpu, mv.to_gpu, mv.for_dst_server, mv.bytes] for mv in moves]
        assert got == c["moves"]
    with pytest.raises(fb.ValidationError):
        fb.balance_senders(fb.TileView(0, 0, np.zeros((2, 2), np.int64)))


@pytest.mark.gpu
def test_strip_and_sort_match_reference():
    import paper_2505_09764_b200 as fb

    g = _golden()
    for c in g["strip"]:
        stages, aux = _as_stages(c["stages"]), np.array(c["aux"], np.int64)
        if c["stripped"] == "error":
            with pytest.raises(fb.InternalInvariantError):
                fb.strip_auxiliary(stages, aux)
            continue
        assert _plain(fb.strip_auxiliary(stages, aux)) == c["stripped"]
    for c in g["sort"]:
        assert _plain(fb.sort_stages_ascending(_as_stages(c["stages"]))) == c["sorted"]
