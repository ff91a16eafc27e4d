"""GPU parity of the bank-balanced CBSR copy (include/maxk.h maxk_topk_cbsr_banked).

A CBSR row is k (value, column) entries (Fig. 4); the aggregation needs the columns of a row distinct,
not ascending.  The banked copy holds the same entries as the oracle's CBSR in the order the header defines (even
columns ascending from the front of the rank list Q, odd columns ascending from its back), which the forward's
NC = 16 row buffers read with a bank conflict only per same-parity pair (t, t + k/2).  Bar: the column-ordered
outputs are bit-identical to maxk_topk_cbsr and the oracle; the banked copy is exactly the header's permutation of
the oracle's row (checked here by an independent restatement of Q); Y = A · CBSR (Eq. 3 left) read
from it meets the north-star row tolerance against the fp64 oracle on both forward layouts.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_08656_b200 import maxk
from test_gpu_parity import _cuda, _graph_with_hubs, assert_rows_close

pytestmark = pytest.mark.gpu


def q_list(k):
    """The header's rank list: positions 4p+e for e = 0..3 and p < k/8, then 4p+e for e = 3..0 and k/8 <= p < k/4."""
    first = [4 * p + e for e in range(4) for p in range(k // 8)]
    second = [4 * p + e for e in (3, 2, 1, 0) for p in range(k // 8, k // 4)]
    return first + second


def expected_banked(rd, ri):
    """The oracle's CBSR rows (ascending columns) permuted into the banked order."""
    n, k = ri.shape
    q = np.array(q_list(k))
    bd = np.empty_like(rd)
    bi = np.empty_like(ri)
    for r in range(n):
        ev = np.flatnonzero(ri[r] % 2 == 0)
        od = np.flatnonzero(ri[r] % 2 == 1)
        pos = np.concatenate([q[: ev.size], q[::-1][: od.size]])
        src = np.concatenate([ev, od])
        bd[r, pos] = rd[r, src]
        bi[r, pos] = ri[r, src]
    return bd, bi


def test_q_list_is_a_permutation_pairing_halves():
    for k in (32, 64, 128):
        q = q_list(k)
        assert sorted(q) == list(range(k))
        # the first k/2 ranks fill the first half, the rest the second; the ranks next to the middle (where an
        # unbalanced row's surplus lands from either side) are group 3 (t % 4 == 3)
        assert all(t < k // 2 for t in q[: k // 2]) and all(t >= k // 2 for t in q[k // 2:])
        L = k // 8
        assert all(q[k // 2 + r] % 4 == 3 and q[k // 2 - 1 - r] % 4 == 3 for r in range(L))


@pytest.mark.parametrize("h", [128, 256, 384, 512])
@pytest.mark.parametrize("k", [32, 64, 128])
@pytest.mark.parametrize("gen", ["normal", "quantized", "special"])
def test_topk_banked_bit_exact(h, k, gen):
    if k > h:
        pytest.skip("k > h")
    n = 1537  # ragged vs the 8-row CTAs
    x = {"normal": synth.normal_f32, "quantized": synth.quantized_f32, "special": synth.special_f32}[gen]((n, h), h + k)
    xd = _cuda(x)
    d, i, bd, bi = maxk.maxk_topk_cbsr_banked(xd, k)
    d0, i0 = maxk.maxk_topk_cbsr(xd, k)
    assert torch.equal(d, d0) and torch.equal(i, i0)  # the column-ordered CBSR is unchanged
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i.cpu().numpy().astype(np.int64), ri)
    ebd, ebi = expected_banked(rd, ri)
    assert np.array_equal(bi.cpu().numpy().astype(np.int64), ebi)
    assert np.array_equal(bd.cpu().numpy().view(np.uint32), ebd.view(np.uint32))


@pytest.mark.parametrize("k", [32, 64, 128])
def test_banked_pairs_conflict_only_when_unbalanced(k):
    """The property the order exists for: among the pairs (t, t + k/2) exactly |n_even - k/2| have equal parity,
    and they sit in group e = 3 (t % 4 == 3) while there are at most k/8 of them."""
    h = 256
    x = synth.normal_f32((4000, h), 7 + k)
    _, _, _, bi = maxk.maxk_topk_cbsr_banked(_cuda(x), k)
    bi = bi.cpu().numpy().astype(np.int64)
    par = bi % 2
    same = par[:, : k // 2] == par[:, k // 2:]
    n_even = (par == 0).sum(axis=1)
    assert np.array_equal(same.sum(axis=1), np.abs(n_even - k // 2))
    t = np.arange(k // 2)[None, :]
    small = np.abs(n_even - k // 2) <= k // 8
    assert np.all((t % 4 == 3) | ~same[small])


@pytest.mark.parametrize("fwd_path", ["0", "2"], ids=["fwd_int", "fwd_rep"])
@pytest.mark.parametrize("h,k", [(256, 32), (256, 64), (256, 128), (128, 32), (512, 64), (384, 128)])
@pytest.mark.parametrize("use_plan", [True, False])
def test_fwd_from_banked_copy(h, k, use_plan, fwd_path, monkeypatch):
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    n_rows, n_cols = 700, 900
    g = _graph_with_hubs(n_rows, n_cols, seed=h + 5 * k)
    x = synth.normal_f32((n_cols, h), h * 3 + k)
    rp, ci, va = _cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val)
    nnz = int(g.row_ptr[-1])
    _, _, bd, bi = maxk.maxk_topk_cbsr_banked(_cuda(x), k)
    plan = maxk.maxk_plan_create(rp, h, k) if use_plan else None
    y = maxk.maxk_spgemm_fwd(rp, ci, va, n_cols, nnz, bd, bi, h, plan=plan)
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y.cpu().numpy(), oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y banked")


@pytest.mark.parametrize("fwd_path", ["1", "2"], ids=["policy", "fwd_rep"])
@pytest.mark.parametrize("k", [32, 64])
def test_fwd_banked_degree_sweep(k, fwd_path, monkeypatch):
    """Rows of every degree 0..320 (every tail of the long-unit pipeline, both sides of the grouped short-row
    threshold), duplicate edges (the same CBSR row twice in one warp step) and negative weights."""
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    h, n_cols = 256, 1200
    rng = np.random.default_rng(300 + k)
    degs = np.concatenate([np.arange(321), rng.integers(0, 321, size=200)])
    rng.shuffle(degs)
    row_ptr = np.zeros(degs.size + 1, np.int64)
    np.cumsum(degs, out=row_ptr[1:])
    col = rng.integers(0, n_cols, size=int(row_ptr[-1])).astype(np.int32)
    col[1::7] = col[::7][: col[1::7].size]  # consecutive duplicates
    val = rng.standard_normal(col.size).astype(np.float32)
    x = synth.normal_f32((n_cols, h), k + 91)
    rp, ci, va = _cuda(row_ptr), _cuda(col), _cuda(val)
    _, _, bd, bi = maxk.maxk_topk_cbsr_banked(_cuda(x), k)
    plan = maxk.maxk_plan_create(rp, h, k)
    y = maxk.maxk_spgemm_fwd(rp, ci, va, n_cols, int(row_ptr[-1]), bd, bi, h, plan=plan).cpu().numpy()
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y, oracle.spgemm_fwd(row_ptr, col, val, rd, ri, h), what="Y banked sweep")


@pytest.mark.parametrize("banked_env", ["2", "0"], ids=["banked", "column"])
@pytest.mark.parametrize("k", [32, 64])
def test_layer_pass_both_orders(k, banked_env, monkeypatch):
    """MaxkAggregation (the layer path bench.py times) with the banked copy forced on (the default where the
    forward uses its NC = 16 buffers) and off: the user-visible CBSR stays in column order, Y and dXs meet the bar
    either way."""
    monkeypatch.setenv("MAXK_BANKED", banked_env)
    from test_gpu_parity import run_gpu
    h = 256
    g = _graph_with_hubs(700, 900, seed=k + 11)
    x = synth.normal_f32((900, h), k + 12)
    dy = synth.normal_f32((700, h), k + 13)
    d, i, y, dxs, _ = run_gpu(g, x, dy, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri) and np.array_equal(d.view(np.uint32), rd.view(np.uint32))
    assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")


def test_layer_falls_back_to_column_order_for_unaligned_x(monkeypatch):
    monkeypatch.setenv("MAXK_BANKED", "2")
    from paper_2312_08656_b200.layer import MaxkAggregation
    h, k = 256, 32
    g = _graph_with_hubs(300, 400, seed=19)
    x = synth.normal_f32((400, h), 20)
    big = torch.zeros((400, h + 1), device="cuda")
    big[:, 1:] = _cuda(x)
    agg = MaxkAggregation(_cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val), g.n_cols, h, k)
    assert agg.sp_bdata is not None
    rd, ri = oracle.topk_cbsr(x, k)
    ref = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h)
    for xin, stale in ((big[:, 1:], True), (_cuda(x), False)):
        agg.topk(xin)
        assert agg._banked_stale == stale
        assert_rows_close(agg.forward().cpu().numpy(), ref, what="Y")
    agg.close()


def test_banked_argument_errors():
    lib = maxk.load()
    x = torch.zeros((16, 256), device="cuda")
    sd = torch.empty((16, 16), device="cuda")
    si = torch.empty((16, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(maxk.MaxkError):  # k = 16: no banked order (the pair layout serves k <= 16)
        maxk.maxk_topk_cbsr_banked(x, 16, sd, si, sd.clone(), si.clone())
    with pytest.raises(maxk.MaxkError):  # h = 100: no float4 top-k
        maxk.maxk_topk_cbsr_banked(torch.zeros((16, 100), device="cuda"), 32)
    d = torch.empty((16, 32), device="cuda")
    i = torch.empty((16, 32), dtype=torch.uint8, device="cuda")
    N = ctypes.c_void_p(0)
    assert lib.maxk_topk_cbsr_banked(x.data_ptr(), 16, 256, 256, 32, 1, d.data_ptr(), i.data_ptr(), N, N, None) == 1
    assert lib.maxk_topk_cbsr_banked(x.data_ptr(), 0, 256, 256, 32, 1, N, N, N, N, None) == 0  # empty: no-op
