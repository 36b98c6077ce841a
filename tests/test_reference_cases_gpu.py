"""The reference's own unit cases for the hot path, restated against the
B200 API (every call below runs the device kernels).

Each test names the tiersched test it mirrors (tests/test_birkhoff.py,
tests/test_balance.py of the reference package); the inputs and expected
values are the reference's, the code is this suite's.  Property cases use
seeded numpy instances instead of hypothesis strategies.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2505_09764_b200 as fb
from paper_2505_09764_b200 import workloads

pytestmark = pytest.mark.gpu

# hand instance of the reference suite (tests/_util.py:103-109)
HAND3 = np.array([[0, 5, 3], [1, 0, 4], [6, 2, 0]], np.int64)


def _rebuild(stages, n, use_weight=False):
    """Sum of the stages' edges as an n x n matrix (weight or edge bytes)."""
    out = np.zeros((n, n), np.int64)
    for st in stages:
        for u, v, b in st.edges:
            out[u, v] += st.weight if use_weight else b
    return out


def _ds_matrix(rng, n, terms, wmax=40):
    """Doubly stochastic integer matrix: a sum of weighted permutations."""
    out = np.zeros((n, n), np.int64)
    for _ in range(terms):
        out[np.arange(n), rng.permutation(n)] += int(rng.integers(1, wmax + 1))
    return out


# ---- embedding (test_birkhoff.py TestEmbed) --------------------------------

def test_embed_diagonal_padding_when_forced():
    # server 0 neither sends nor receives: its deficit can only sit on the
    # diagonal (test_birkhoff.py:50-60)
    s = fb.ServerMatrix(np.array([[0, 0, 0], [0, 0, 5], [0, 5, 0]], np.int64))
    emb, aux = fb.embed_doubly_stochastic(s)
    assert aux[0, 0] == 5
    assert (emb.sum(axis=1) == 5).all() and (emb.sum(axis=0) == 5).all()


def test_embed_zero_matrix():
    emb, aux = fb.embed_doubly_stochastic(fb.ServerMatrix(np.zeros((3, 3), np.int64)))
    assert emb.sum() == 0 and aux.sum() == 0


def _seeded_server(seed, n, modulus=997):
    """The reference suite's seeded server matrix (tests/_util.py:34-39):
    rng.stream(seed, n*n) mod 997, zero diagonal."""
    t = (workloads.stream(seed, n * n) % np.uint64(modulus)).astype(np.int64).reshape(n, n)
    np.fill_diagonal(t, 0)
    return fb.ServerMatrix(t)


def test_embed_equalizes_and_keeps_demand():
    # test_birkhoff.py:40-48 on the suite's seeded server matrices
    for seed in range(12):
        s = _seeded_server(seed, 2 + seed % 6)
        emb, aux = fb.embed_doubly_stochastic(s)
        common = fb.max_rc(s)
        assert (emb.sum(axis=1) == common).all() and (emb.sum(axis=0) == common).all()
        assert (aux >= 0).all()
        assert np.array_equal(emb - aux, s.off_diagonal())


# ---- perfect matching (test_birkhoff.py TestPerfectMatching) ---------------

def test_matching_permutation_support():
    sup = np.zeros((3, 3), bool)
    for u, v in [(0, 2), (1, 0), (2, 1)]:
        sup[u, v] = True
    assert fb.find_perfect_matching(sup) == {0: 2, 1: 0, 2: 1}


def test_matching_needs_augmenting_path():
    sup = np.array([[1, 1, 0], [1, 0, 0], [0, 1, 1]], bool)
    mt = fb.find_perfect_matching(sup)
    assert sorted(mt) == [0, 1, 2] and sorted(mt.values()) == [0, 1, 2]
    assert all(sup[u, v] for u, v in mt.items())


def test_matching_absent_raises():
    sup = np.array([[1, 0, 0], [1, 0, 0], [1, 1, 1]], bool)
    with pytest.raises(fb.InternalInvariantError):
        fb.find_perfect_matching(sup)


def test_matching_full_support_pins_anti_diagonal():
    sup = np.ones((4, 4), bool)
    assert fb.find_perfect_matching(sup) == {0: 3, 1: 2, 2: 1, 3: 0}


# ---- decompose (test_birkhoff.py TestDecompose) ----------------------------

@pytest.mark.parametrize("bad, needle", [
    (np.zeros((2, 3), np.int64), "square"),
    (np.zeros((2, 2), np.float64), "integer"),
    (np.array([[1, -1], [-1, 1]], np.int64), "non-negative"),
    (np.array([[2, 0], [0, 1]], np.int64), "equal row"),
])
def test_decompose_input_validation(bad, needle):
    with pytest.raises(fb.ValidationError, match=needle):
        fb.decompose(bad)


def test_decompose_zero_matrix_gives_no_stages():
    assert fb.decompose(np.zeros((3, 3), np.int64)) == []


def test_decompose_identity_times_weight():
    stages = fb.decompose(7 * np.eye(4, dtype=np.int64))
    assert len(stages) == 1 and stages[0].weight == 7
    assert stages[0].matching == {0: 0, 1: 1, 2: 2, 3: 3}


def test_decompose_one_by_one():
    stages = fb.decompose(np.array([[5]], np.int64))
    assert len(stages) == 1 and stages[0].weight == 5 and stages[0].edges == ((0, 0, 5),)
    assert fb.decompose(np.array([[0]], np.int64)) == []


def test_decompose_exact_reconstruction_and_determinism():
    # test_birkhoff.py:124-141: reconstruction, the n^2 - 2n + 2 bound,
    # positive weights summing to the common row sum, full permutations
    rng = np.random.default_rng(2024)
    for _ in range(60):
        n = int(rng.integers(2, 8))
        e = _ds_matrix(rng, n, int(rng.integers(1, 7)))
        stages = fb.decompose(e)
        assert np.array_equal(_rebuild(stages, n, use_weight=True), e)
        assert len(stages) <= n * n - 2 * n + 2
        assert all(st.weight > 0 for st in stages)
        assert sum(st.weight for st in stages) == int(e.sum(axis=1)[0])
        assert all(len(st.edges) == n for st in stages)
        assert fb.decompose(e.copy()) == stages


# ---- strip / sort (test_birkhoff.py TestStrip, TestSortStages) -------------

def test_strip_aux_charged_before_real():
    P = fb.PermutationStage
    stages = [P(weight=3, edges=((0, 0, 3), (1, 1, 3))), P(weight=2, edges=((0, 1, 2), (1, 0, 2)))]
    out = fb.strip_auxiliary(stages, np.array([[3, 1], [0, 0]], np.int64))
    assert len(out) == 2
    assert out[0].edges == ((1, 1, 3),) and out[0].weight == 3
    assert out[1].edges == ((0, 1, 1), (1, 0, 2))


def test_strip_pure_aux_stage_disappears():
    P = fb.PermutationStage
    stages = [P(weight=4, edges=((0, 1, 4), (1, 0, 4)))]
    assert fb.strip_auxiliary(stages, np.array([[0, 4], [4, 0]], np.int64)) == []


def test_strip_leftover_aux_is_loud():
    P = fb.PermutationStage
    stages = [P(weight=1, edges=((0, 0, 1), (1, 1, 1)))]
    with pytest.raises(fb.InternalInvariantError):
        fb.strip_auxiliary(stages, np.array([[5, 0], [0, 0]], np.int64))


def test_strip_covers_exactly_the_real_bytes():
    # test_birkhoff.py:170-183: half of a DS matrix as aux, half as demand
    rng = np.random.default_rng(77)
    for _ in range(40):
        n = int(rng.integers(2, 7))
        e = _ds_matrix(rng, n, int(rng.integers(1, 7)))
        real = e // 2
        out = fb.strip_auxiliary(fb.decompose(e), e - real)
        assert np.array_equal(_rebuild(out, n), real)
        for st in out:
            assert st.edges and all(0 < b <= st.weight for _, _, b in st.edges)


def test_sort_ascending_with_edge_tiebreak():
    P = fb.PermutationStage
    a = P(weight=2, edges=((1, 0, 2),))
    b = P(weight=1, edges=((0, 1, 1),))
    c = P(weight=2, edges=((0, 1, 2),))
    assert fb.sort_stages_ascending([a, b, c]) == [b, c, a]


def test_sort_stable_for_full_ties():
    P = fb.PermutationStage
    a = P(weight=2, edges=((0, 1, 2), (1, 0, 2)))
    b = P(weight=2, edges=((0, 1, 2), (2, 2, 2)))
    assert fb.sort_stages_ascending([a, b]) == [a, b]
    assert fb.sort_stages_ascending([b, a]) == [b, a]


# ---- server matrices (test_birkhoff.py TestServerMatrixDecomposition) ------

def test_server_decomposition_hand_instance():
    s = fb.ServerMatrix(HAND3.copy())
    d = fb.decompose_server_matrix(s)
    assert d.common_sum == 8 and sum(st.weight for st in d.stages) == 8
    assert np.array_equal(_rebuild(list(d.stages), 3, True), s.off_diagonal() + d.aux)


def test_server_decomposition_random_instances_reconstruct():
    # test_birkhoff.py:210-224
    for seed in range(25):
        n = 2 + seed % 7
        s = _seeded_server(seed, n)
        d = fb.decompose_server_matrix(s)
        assert np.array_equal(_rebuild(list(d.stages), n, True), s.off_diagonal() + d.aux)
        out = fb.strip_auxiliary(list(d.stages), d.aux)
        assert np.array_equal(_rebuild(out, n), s.off_diagonal())


# ---- sender balancing (test_balance.py TestBalanceSenders) -----------------

def _cross(tile):
    return fb.TileView(src_server=0, dst_server=1, entries=tile)


def test_balance_single_loaded_row_spreads_out():
    bal, moves = fb.balance_senders(_cross(np.array([[7, 0, 0], [0, 0, 0], [0, 0, 0]], np.int64)))
    assert bal.sum(axis=1).tolist() == [3, 2, 2]
    assert sum(mv.bytes for mv in moves) == 4
    assert bal.sum(axis=0).tolist() == [7, 0, 0]


def test_balance_already_balanced_needs_no_moves():
    tile = np.array([[2, 1], [1, 2]], np.int64)
    bal, moves = fb.balance_senders(_cross(tile))
    assert moves == [] and np.array_equal(bal, tile)


def test_balance_rejects_intra_tile():
    with pytest.raises(fb.ValidationError):
        fb.balance_senders(fb.TileView(src_server=1, dst_server=1, entries=np.zeros((2, 2), np.int64)))


def test_balance_invariants_on_random_tiles():
    # test_balance.py:63-85: conservation, column preservation, row targets,
    # move volume = row surplus, moves tagged for (server 0 -> server 1)
    rng = np.random.default_rng(5)
    for _ in range(80):
        m = int(rng.integers(2, 7))
        tile = rng.integers(0, 31, size=(m, m)).astype(np.int64)
        bal, moves = fb.balance_senders(_cross(tile.copy()))
        again = fb.balance_senders(_cross(tile.copy()))
        assert np.array_equal(again[0], bal) and again[1] == moves
        total = int(tile.sum())
        base, extra = divmod(total, m)
        expect = [base + 1] * extra + [base] * (m - extra)
        assert int(bal.sum()) == total
        assert np.array_equal(bal.sum(axis=0), tile.sum(axis=0))
        assert bal.sum(axis=1).tolist() == expect and (bal >= 0).all()
        surplus = sum(int(r) - e for r, e in zip(tile.sum(axis=1), expect) if r > e)
        assert sum(mv.bytes for mv in moves) == surplus
        for mv in moves:
            assert mv.server == 0 and mv.for_dst_server == 1
            assert 0 <= mv.from_gpu < m and 0 <= mv.to_gpu < m
