"""Pins for the CPU oracle (oracle/), independent of the oracle's own code.

Each test checks the oracle against something the paper or mathematics fixes: the hand-worked example
(tests/golden/worked_example.json), brute force on tiny inputs, a library routine (numpy dense matmul,
numpy stable argsort, scipy.sparse), closed forms (k=H, A=I, constant rows) and invariants
(adjointness of Eq. 3's forward/backward pair). A plausible slip in the oracle — a dropped term, a
wrong sign or index, a transposed operand, a wrong tie-break — fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")


def _f32(v):
    return np.float32(float(v)) if not isinstance(v, str) else np.float32(float(v))


def _load_golden():
    with open(GOLDEN) as f:
        g = json.load(f)
    X = np.array([[_f32(v) for v in row] for row in g["X"]], dtype=np.float32)
    data = np.array([[_f32(v) for v in row] for row in g["data"]], dtype=np.float32)
    return g, X, data


def _dense_A(row_ptr, col_idx, val, n_cols):
    n = len(row_ptr) - 1
    A = np.zeros((n, n_cols), dtype=np.float64)
    for i in range(n):
        for e in range(row_ptr[i], row_ptr[i + 1]):
            A[i, col_idx[e]] += float(val[e])  # duplicates are summed (reading R12)
    return A


# ------------------------------------------------------------------------------------------------
# hand-worked example (Fig. 6/7 shape dim_origin=6, dim_k=3)
# ------------------------------------------------------------------------------------------------
def test_golden_topk_bits():
    g, X, data_ref = _load_golden()
    data, idx = oracle.topk_cbsr(X, g["k"])
    assert idx.tolist() == g["idx"]
    # bit-exact including the -0.0 kept in row 3 (reading R3)
    assert data.view(np.uint32).tolist() == data_ref.view(np.uint32).tolist()
    assert np.signbit(data[3, 0])


def test_golden_forward_backward_adjoint():
    g, X, _ = _load_golden()
    data, idx = oracle.topk_cbsr(X, g["k"])
    rp = np.array(g["row_ptr"], np.int64)
    ci = np.array(g["col_idx"], np.int32)
    va = np.array(g["val"], np.float32)
    Y = oracle.spgemm_fwd(rp, ci, va, data, idx, g["H"])
    assert np.array_equal(Y, np.array(g["Y"]))
    dY = np.array([[10 * i + c for c in range(g["H"])] for i in range(5)], np.float32)
    dXs = oracle.sspmm_bwd(rp, ci, va, dY, idx)
    assert np.array_equal(dXs, np.array(g["dXs"]))
    assert float((Y * dY).sum()) == g["adjoint_inner_product"]
    assert float((data.astype(np.float64) * dXs).sum()) == g["adjoint_inner_product"]


# ------------------------------------------------------------------------------------------------
# top-k (Eq. 1)
# ------------------------------------------------------------------------------------------------
def test_spec_examples():
    d, i = oracle.topk_cbsr(np.array([[0.9, -0.2, 0.5, 0.1]], np.float32), 2)
    assert i.tolist() == [[0, 2]] and d.tolist() == [[np.float32(0.9), np.float32(0.5)]]
    x = np.full((3, 7), 0.3, np.float32)
    _, i = oracle.topk_cbsr(x, 2)
    assert i.tolist() == [[0, 1]] * 3


def test_k_equals_h_is_identity():
    x = synth.special_f32((50, 33), seed=5)
    d, i = oracle.topk_cbsr(x, 33)
    assert np.array_equal(i, np.tile(np.arange(33, dtype=np.int32), (50, 1)))
    assert np.array_equal(d.view(np.uint32), x.view(np.uint32))


def _brute_force_topk(v, k):
    """The unique size-k subset S with: every s in S ranks before every u not in S."""
    h = len(v)
    winners = []
    for S in itertools.combinations(range(h), k):
        Sset = set(S)
        ok = all((v[s] > v[u]) or (v[s] == v[u] and s < u) for s in S for u in range(h) if u not in Sset)
        if ok:
            winners.append(list(S))
    assert len(winners) == 1
    return winners[0]


def test_topk_brute_force_small():
    rng = np.random.default_rng(11)
    for trial in range(300):
        h = int(rng.integers(1, 9))
        k = int(rng.integers(1, h + 1))
        if trial % 3 == 0:
            v = synth.quantized_f32((1, h), seed=trial)
        elif trial % 3 == 1:
            v = synth.special_f32((1, h), seed=trial)
        else:
            v = rng.standard_normal((1, h)).astype(np.float32)
        d, i = oracle.topk_cbsr(v, k)
        assert i[0].tolist() == _brute_force_topk([float(a) for a in v[0]], k)


def test_topk_matches_numpy_stable_argsort():
    # library routine: stable argsort of -x orders by value desc, ties (incl. -0.0 == +0.0) by index
    for seed, gen in [(1, synth.quantized_f32), (2, synth.special_f32), (3, synth.normal_f32)]:
        x = gen((400, 256), seed) if gen is not synth.normal_f32 else gen((400, 256), seed)
        for k in (1, 8, 32, 100, 256):
            d, i = oracle.topk_cbsr(x, k)
            ref = np.sort(np.argsort(-x, axis=1, kind="stable")[:, :k], axis=1)
            assert np.array_equal(i, ref)
            assert np.array_equal(d.view(np.uint32), np.take_along_axis(x, ref, 1).view(np.uint32))


def test_topk_invariants():
    x = synth.quantized_f32((300, 64), seed=9)
    k = 13
    d, i = oracle.topk_cbsr(x, k)
    for r in range(x.shape[0]):
        assert np.all(np.diff(i[r]) > 0) and i[r, 0] >= 0 and i[r, -1] < 64
        sel = set(i[r].tolist())
        mn = min(x[r, c] for c in sel)
        for u in range(64):
            if u not in sel:
                assert x[r, u] <= mn
                if x[r, u] == mn:
                    assert all(u > c for c in sel if x[r, c] == mn)


def test_topk_rejects_nan_and_bad_k():
    x = np.zeros((2, 4), np.float32)
    x[1, 2] = np.nan
    with pytest.raises(ValueError):
        oracle.topk_cbsr(x, 2)
    with pytest.raises(ValueError):
        oracle.topk_cbsr(np.zeros((2, 4), np.float32), 5)
    with pytest.raises(ValueError):
        oracle.topk_cbsr(np.zeros((2, 4), np.float32), 0)


# ------------------------------------------------------------------------------------------------
# forward SpGEMM and backward SSpMM (Eq. 3)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(20))
def test_fwd_bwd_vs_dense_brute_force(seed):
    rng = np.random.default_rng(seed)
    n, nc = int(rng.integers(1, 40)), int(rng.integers(1, 40))
    h = int(rng.choice([4, 8, 16, 32]))
    k = int(rng.integers(1, h + 1))
    g = synth.random_csr(n, nc, avg_deg=3.0, seed=seed, duplicates=(seed % 2 == 0))
    x = rng.standard_normal((nc, h)).astype(np.float32)
    dy = rng.standard_normal((n, h)).astype(np.float32)
    data, idx = oracle.topk_cbsr(x, k)
    A = _dense_A(g.row_ptr, g.col_idx, g.val, nc)
    D = np.zeros((nc, h))
    for j in range(nc):
        D[j, idx[j]] = data[j]
    Y = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, data, idx, h)
    np.testing.assert_allclose(Y, A @ D, rtol=1e-12, atol=1e-12)
    G = A.T @ dy.astype(np.float64)
    dXs = oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, idx)
    np.testing.assert_allclose(dXs, np.take_along_axis(G, idx.astype(np.int64), 1), rtol=1e-12, atol=1e-12)
    # adjointness <A·D, dY> = <D, A^T dY> restricted to the pattern
    lhs = float((Y * dy).sum())
    rhs = float((data.astype(np.float64) * dXs).sum())
    assert abs(lhs - rhs) <= 1e-9 * (1 + abs(lhs))


def test_k_equals_h_reduces_to_spmm_scipy():
    g = synth.power_law_graph(600, 6000, seed=77)
    h = 24
    x = synth.normal_f32((600, h), seed=3)
    dy = synth.normal_f32((600, h), seed=4)
    data, idx = oracle.topk_cbsr(x, h)
    A = sp.csr_matrix((g.val.astype(np.float64), g.col_idx, g.row_ptr), shape=(600, 600))
    Y = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, data, idx, h)
    np.testing.assert_allclose(Y, A @ x.astype(np.float64), rtol=1e-12, atol=1e-12)
    dXs = oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, idx)
    np.testing.assert_allclose(dXs, A.T @ dy.astype(np.float64), rtol=1e-12, atol=1e-12)


def test_identity_adjacency():
    n, h, k = 50, 16, 5
    x = synth.normal_f32((n, h), seed=8)
    dy = synth.normal_f32((n, h), seed=9)
    data, idx = oracle.topk_cbsr(x, k)
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    va = np.ones(n, np.float32)
    Y = oracle.spgemm_fwd(rp, ci, va, data, idx, h)
    assert np.array_equal(Y, oracle.densify(data, idx, h))
    dXs = oracle.sspmm_bwd(rp, ci, va, dy, idx)
    assert np.array_equal(dXs, np.take_along_axis(dy, idx.astype(np.int64), 1).astype(np.float64))


def test_mean_aggregator_of_identical_rows():
    # A' = D^-1 A (SAGE mean): identical densified rows v give Y[i] = v on deg>0 rows
    g = synth.random_csr(80, 80, avg_deg=6.0, seed=3, weights="mean")
    h, k = 32, 4
    row = np.zeros((1, h), np.float32)
    row[0, [3, 9, 20, 31]] = [2.0, 1.0, 0.5, 4.0]  # the 4 positives are the top-4
    x = np.repeat(row, 80, 0)
    data, idx = oracle.topk_cbsr(x, k)
    Y = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, data, idx, h)
    deg = np.diff(g.row_ptr)
    np.testing.assert_allclose(Y[deg > 0], np.repeat(row.astype(np.float64), int((deg > 0).sum()), 0),
                               rtol=1e-6)
    assert np.all(Y[deg == 0] == 0)


def test_transpose_matches_scipy():
    g = synth.random_csr(70, 55, avg_deg=5.0, seed=12)
    t_ptr, t_row, t_val = oracle.transpose(g.row_ptr, g.col_idx, g.val, 55)
    At = sp.csr_matrix((g.val, g.col_idx, g.row_ptr), shape=(70, 55)).T.tocsr()
    At.sort_indices()
    assert np.array_equal(t_ptr, At.indptr)
    assert np.array_equal(t_row, At.indices)
    assert np.array_equal(t_val, At.data)


def test_row_subsets_match_full():
    g = synth.power_law_graph(500, 4000, seed=21)
    h, k = 32, 8
    x = synth.normal_f32((500, h), seed=1)
    dy = synth.normal_f32((500, h), seed=2)
    data, idx = oracle.topk_cbsr(x, k)
    rows = np.array([0, 7, 499, 250, 7], np.int64)
    Y = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, data, idx, h)
    assert np.array_equal(oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, data, idx, h, rows=rows), Y[rows])
    dX = oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, idx)
    assert np.array_equal(oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, idx, rows=rows), dX[rows])


def test_linear_hand_example():
    # Eq. 1's argument X·W + b on a 2x3 · 3x2 example worked by hand
    x = np.array([[1.0, 2.0, -1.0], [0.5, 0.0, 4.0]])
    w = np.array([[1.0, 0.0], [2.0, -1.0], [0.0, 3.0]])       # f x h
    b = np.array([0.25, -0.5])
    z = oracle.linear(x, w.T, b)
    assert np.array_equal(z, np.array([[5.25, -5.5], [0.75, 11.5]]))
