"""GPU parity of the CBSR pair layout (include/maxk.h maxk_topk_cbsr_pairs / maxk_spgemm_fwd_pairs).

The pair layout is a B200-specific companion of the two-block CBSR for k in {8, 16}: {value bits, column} per entry,
so one 128-byte line holds a whole gathered row.  Bar: the pairs are a bit-exact re-layout of the oracle's CBSR
(PAPER.md:326), and Y = A · CBSR (Eq. 3 left) from them meets the north-star row tolerance against
the fp64 oracle and is bit-identical to the two-block forward (same kernel, same summation order).  The k = 16
balanced pair order (maxk_topk_cbsr_pairs_banked) is checked against an independent restatement of its rule.
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


def _split(pairs: torch.Tensor):
    p = pairs.cpu().numpy()
    return p[..., 0].view(np.uint32), p[..., 1].astype(np.int64)


@pytest.mark.parametrize("h", [128, 256, 384, 512])
@pytest.mark.parametrize("k", [8, 16])
@pytest.mark.parametrize("gen", ["normal", "quantized", "special"])
def test_topk_pairs_bit_exact(h, k, gen):
    n = 1537  # ragged vs the 8-row CTAs
    x = {"normal": synth.normal_f32, "quantized": synth.quantized_f32, "special": synth.special_f32}[gen]((n, h), h + k)
    xd = _cuda(x)
    d, i, p = maxk.maxk_topk_cbsr_pairs(xd, k)
    d0, i0 = maxk.maxk_topk_cbsr(xd, k)
    rd, ri = oracle.topk_cbsr(x, k)
    bits, cols = _split(p)
    assert np.array_equal(cols, ri) and np.array_equal(bits, rd.view(np.uint32))
    assert np.array_equal(i.cpu().numpy().astype(np.int64), ri)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), rd.view(np.uint32))
    assert torch.equal(d, d0) and torch.equal(i, i0)


@pytest.mark.parametrize("h,k", [(256, 8), (256, 16), (128, 8), (512, 16), (384, 16)])
@pytest.mark.parametrize("use_plan", [True, False])
def test_fwd_pairs_parity(h, k, use_plan):
    n_rows, n_cols = 700, 900
    g = _graph_with_hubs(n_rows, n_cols, seed=h + 3 * k)
    x = synth.normal_f32((n_cols, h), h * 5 + k)
    rp, ci, va = _cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val)
    nnz = int(g.row_ptr[-1])
    sd, si, sp = maxk.maxk_topk_cbsr_pairs(_cuda(x), k)
    plan = maxk.maxk_plan_create(rp, h, k) if use_plan else None
    y = maxk.maxk_spgemm_fwd_pairs(rp, ci, va, n_cols, nnz, sp, h, plan=plan)
    y2 = maxk.maxk_spgemm_fwd(rp, ci, va, n_cols, nnz, sd, si, h, plan=plan)
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y.cpu().numpy(), oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y pairs")
    assert torch.equal(y, y2)  # same kernel and lane mapping: bit-identical to the two-block forward


@pytest.mark.parametrize("k", [8, 16])
def test_fwd_pairs_degree_sweep(k):
    """Rows of every degree 0..320 (every tail of the long-unit pipeline, both sides of the grouped short-row
    threshold), duplicates and negative weights."""
    h, n_cols = 256, 1200
    rng = np.random.default_rng(100 + k)
    degs = np.concatenate([np.arange(321), rng.integers(0, 321, size=200)])
    rng.shuffle(degs)
    row_ptr = np.zeros(degs.size + 1, np.int64)
    np.cumsum(degs, out=row_ptr[1:])
    col = rng.integers(0, n_cols, size=int(row_ptr[-1])).astype(np.int32)
    val = rng.standard_normal(col.size).astype(np.float32)
    x = synth.normal_f32((n_cols, h), k + 77)
    rp, ci, va = _cuda(row_ptr), _cuda(col), _cuda(val)
    _, _, sp = maxk.maxk_topk_cbsr_pairs(_cuda(x), k)
    plan = maxk.maxk_plan_create(rp, h, k)
    y = maxk.maxk_spgemm_fwd_pairs(rp, ci, va, n_cols, int(row_ptr[-1]), sp, h, plan=plan).cpu().numpy()
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y, oracle.spgemm_fwd(row_ptr, col, val, rd, ri, h), what="Y pairs sweep")


@pytest.mark.parametrize("pairs_env", ["1", "0"], ids=["pairs", "two_block"])
@pytest.mark.parametrize("k", [8, 16])
def test_layer_pass_both_layouts(k, pairs_env, monkeypatch):
    """MaxkAggregation (the layer path bench.py times) with the pair layout on (default for k in {8, 16}) and off."""
    monkeypatch.setenv("MAXK_PAIRS", pairs_env)
    from test_gpu_parity import run_gpu
    h = 256
    g = _graph_with_hubs(700, 900, seed=k + 1)
    x = synth.normal_f32((900, h), k + 2)
    dy = synth.normal_f32((700, h), k + 3)
    d, i, y, dxs, _ = run_gpu(g, x, dy, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri) and np.array_equal(d.view(np.uint32), rd.view(np.uint32))
    assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")


def test_pairs_argument_errors():
    lib = maxk.load()
    x = torch.zeros((16, 256), device="cuda")
    sd = torch.empty((16, 32), device="cuda")
    si = torch.empty((16, 32), dtype=torch.uint8, device="cuda")
    sp = torch.empty((16, 32, 2), dtype=torch.int32, device="cuda")
    with pytest.raises(maxk.MaxkError):  # k = 32: a row is two lines either way -> UNSUPPORTED
        maxk.maxk_topk_cbsr_pairs(x, 32, sd, si, sp)
    with pytest.raises(maxk.MaxkError):  # h = 100: no float4 top-k
        maxk.maxk_topk_cbsr_pairs(torch.zeros((16, 100), device="cuda"), 8)
    P = ctypes.c_void_p(sp.data_ptr() + 8)  # misaligned pair block
    assert lib.maxk_topk_cbsr_pairs(x.data_ptr(), 16, 256, 256, 8, 1, sd.data_ptr(), si.data_ptr(), P, None) == 1
    Q = ctypes.c_void_p(0x1000)
    assert lib.maxk_spgemm_fwd_pairs(Q, Q, Q, 4, 4, 8, Q, 256, 32, Q, 256, None, None) == 2
    assert lib.maxk_spgemm_fwd_pairs(Q, Q, Q, 4, 4, 8, P, 256, 8, Q, 256, None, None) == 1


def test_layer_falls_back_to_two_blocks_for_unaligned_x():
    """MaxkAggregation keeps working when x cannot feed the pair-writing top-k (rows not 16-byte aligned): the
    forward then reads the two-block CBSR, and a later aligned full pass returns to the pair layout."""
    from paper_2312_08656_b200.layer import MaxkAggregation
    h, k = 256, 8
    g = _graph_with_hubs(300, 400, seed=9)
    x = synth.normal_f32((400, h), 10)
    big = torch.zeros((400, h + 1), device="cuda")
    big[:, 1:] = _cuda(x)
    x_unaligned = big[:, 1:]  # 4-byte offset rows
    agg = MaxkAggregation(_cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val), g.n_cols, h, k)
    rd, ri = oracle.topk_cbsr(x, k)
    ref = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h)
    for xin in (x_unaligned, _cuda(x)):
        agg.topk(xin)
        y = agg.forward().cpu().numpy()
        assert_rows_close(y, ref, what="Y")
    assert agg.sp_pairs is not None and not agg._pairs_stale
    agg.close()


@pytest.mark.parametrize("h", [128, 256, 512])
@pytest.mark.parametrize("gen", ["normal", "quantized", "special"])
def test_topk_pairs_banked_order(h, gen):
    """maxk_topk_cbsr_pairs_banked (k = 16): sp_data / sp_idx as maxk_topk_cbsr; the pairs are the oracle's row
    permuted by the header's mod-4-balanced rule (restated independently in balanced_pair_order)."""
    k, n = 16, 1537
    x = {"normal": synth.normal_f32, "quantized": synth.quantized_f32, "special": synth.special_f32}[gen]((n, h), h + 5)
    xd = _cuda(x)
    d, i, p = maxk.maxk_topk_cbsr_pairs(xd, k, banked=True)
    d0, i0 = maxk.maxk_topk_cbsr(xd, k)
    assert torch.equal(d, d0) and torch.equal(i, i0)
    rd, ri = oracle.topk_cbsr(x, k)
    bits, cols = _split(p)
    src = balanced_pair_order(ri)
    assert np.array_equal(cols, np.take_along_axis(ri, src, 1))
    assert np.array_equal(bits, np.take_along_axis(rd.view(np.uint32), src, 1))


def balanced_pair_order(ri):
    """src[r, pos] = column-order index the k = 16 balanced pair layout puts at pos: class m = c mod 4 takes position
    2 (pi + 2m) + e of the sets j = (e, pi) = (j // 2, j % 2) in order; the entries of a class beyond its fourth, in
    ascending column order, fill the slots deficient classes leave free, set 3 first, then by class."""
    n, k = ri.shape
    src = np.empty((n, k), np.int64)
    for r in range(n):
        cls = [np.flatnonzero(ri[r] % 4 == m) for m in range(4)]
        cnt = [c.size for c in cls]
        surplus = sorted(t for m in range(4) for t in cls[m][4:])
        for m in range(4):
            for j, t in enumerate(cls[m][:4]):
                src[r, 2 * ((j % 2) + 2 * m) + j // 2] = t
        free = [(j, m) for j in (3, 2, 1, 0) for m in range(4) if cnt[m] <= j]
        assert len(free) == len(surplus)
        for t, (j, m) in zip(surplus, free):
            src[r, 2 * ((j % 2) + 2 * m) + j // 2] = t
    return src


@pytest.mark.parametrize("fwd_path", ["0", "2"], ids=["nc_epi", "nc8"])
@pytest.mark.parametrize("use_plan", [True, False])
def test_fwd_pairs_banked_parity(use_plan, fwd_path, monkeypatch):
    """The pair-layout forward from the balanced order, with NC = EPI and NC = 8 row buffers (forced), hub rows
    split into chunks, against the fp64 oracle."""
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    h, k, n_rows, n_cols = 256, 16, 700, 900
    g = _graph_with_hubs(n_rows, n_cols, seed=61)
    x = synth.normal_f32((n_cols, h), 62)
    rp, ci, va = _cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val)
    _, _, sp = maxk.maxk_topk_cbsr_pairs(_cuda(x), k, banked=True)
    plan = maxk.maxk_plan_create(rp, h, k) if use_plan else None
    y = maxk.maxk_spgemm_fwd_pairs(rp, ci, va, n_cols, int(g.row_ptr[-1]), sp, h, plan=plan)
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y.cpu().numpy(), oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")


@pytest.mark.parametrize("fwd_path", ["1", "2"], ids=["policy", "nc8"])
def test_fwd_pairs_banked_degree_sweep(fwd_path, monkeypatch):
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    h, k, n_cols = 256, 16, 1200
    rng = np.random.default_rng(116)
    degs = np.concatenate([np.arange(321), rng.integers(0, 321, size=200)])
    rng.shuffle(degs)
    row_ptr = np.zeros(degs.size + 1, np.int64)
    np.cumsum(degs, out=row_ptr[1:])
    col = rng.integers(0, n_cols, size=int(row_ptr[-1])).astype(np.int32)
    val = rng.standard_normal(col.size).astype(np.float32)
    x = synth.normal_f32((n_cols, h), 93)
    rp, ci, va = _cuda(row_ptr), _cuda(col), _cuda(val)
    _, _, sp = maxk.maxk_topk_cbsr_pairs(_cuda(x), k, banked=True)
    plan = maxk.maxk_plan_create(rp, h, k)
    y = maxk.maxk_spgemm_fwd_pairs(rp, ci, va, n_cols, int(row_ptr[-1]), sp, h, plan=plan).cpu().numpy()
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y, oracle.spgemm_fwd(row_ptr, col, val, rd, ri, h), what="Y balanced pairs sweep")


def test_pairs_banked_rejects_k8():
    x = torch.zeros((16, 256), device="cuda")
    with pytest.raises(maxk.MaxkError):
        maxk.maxk_topk_cbsr_pairs(x, 8, banked=True)
