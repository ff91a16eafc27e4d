"""GPU parity: the CUDA path through the C-ABI against the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star; DESIGN.md §2 "comparison rule"):
  - CBSR sp_idx and sp_data bit-exact (the top-k mask is identical);
  - Y and dXs: every row satisfies max_c |gpu - ref| <= 1e-5 * (1 + max_c |ref|), ref in fp64.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_08656_b200 import maxk
from paper_2312_08656_b200.layer import MaxkAggregation

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_rows_close(gpu: np.ndarray, ref: np.ndarray, tol: float = TOL, what: str = "") -> float:
    """Row-wise bar of the north star; returns the worst err/tol ratio (SURVEY §8(c) c.6 reports it)."""
    gpu = gpu.astype(np.float64)
    assert gpu.shape == ref.shape
    if ref.size == 0:
        return 0.0
    err = np.abs(gpu - ref).max(axis=1)
    bound = tol * (1.0 + np.abs(ref).max(axis=1))
    worst = int(np.argmax(err / bound))
    assert np.all(err <= bound), f"{what}: row {worst} err {err[worst]:.3e} > tol {bound[worst]:.3e}"
    ratio = float(err[worst] / bound[worst])
    print(f"[parity] {what}: {ref.shape[0]} rows, worst err/tol {ratio:.4f}")
    return ratio


def gpu_topk(x: np.ndarray, k: int):
    d, i = maxk.maxk_topk_cbsr(_cuda(x), k)
    torch.cuda.synchronize()
    return d.cpu().numpy(), i.cpu().numpy().astype(np.int32)


# ------------------------------------------------------------------------------------------------
# top-k -> CBSR: bit-exact
# ------------------------------------------------------------------------------------------------
TOPK_CASES = [
    # (h, k, generator)
    (256, 32, "normal"), (256, 8, "normal"), (256, 16, "normal"), (256, 64, "normal"), (256, 1, "normal"),
    (256, 256, "normal"), (256, 32, "quantized"), (256, 32, "special"), (256, 100, "quantized"),
    (64, 8, "normal"), (64, 8, "quantized"), (64, 64, "special"), (128, 5, "special"),
    (100, 7, "quantized"), (33, 33, "special"), (1, 1, "normal"), (300, 30, "normal"), (384, 48, "quantized"),
    (1024, 32, "normal"), (1000, 999, "quantized"), (512, 17, "special"),
]


@pytest.mark.parametrize("h,k,gen", TOPK_CASES)
def test_topk_bit_exact(h, k, gen):
    n = 1537  # ragged vs the 8-row CTAs
    seed = h * 1000 + k
    x = {"normal": lambda: synth.normal_f32((n, h), seed), "quantized": lambda: synth.quantized_f32((n, h), seed),
         "special": lambda: synth.special_f32((n, h), seed)}[gen]()
    d, i = gpu_topk(x, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri)
    assert np.array_equal(d.view(np.uint32), rd.view(np.uint32))


@pytest.mark.parametrize("k", [8, 16, 32, 64])
def test_topk_probe_statistic(k):
    """SPEC.md:544 / PAPER.md:675 ("less than 10 iterations"): the pivot search of the default top-k kernel, on
    N(0,1) rows (the feature map "follows a normal distribution"), H = 256, takes a median of <= 10
    probes per row. The statistic entry point selects exactly what maxk_topk_cbsr selects (bit-exact) and the
    oracle agrees. Exactness never depends on the cap: rows whose probes cannot split exactly k fall back to the
    exact key descent (counted separately)."""
    n, h = 20000, 256
    x = synth.normal_f32((n, h), seed=4242 + k)
    d, i, probes = maxk.maxk_topk_cbsr_probe_stats(_cuda(x), k)
    d2, i2 = maxk.maxk_topk_cbsr(_cuda(x), k)
    torch.cuda.synchronize()
    assert torch.equal(i, i2) and torch.equal(d.view(torch.int32), d2.view(torch.int32))
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i.cpu().numpy().astype(np.int32), ri)
    pr = probes.cpu().numpy()
    exact = pr >= 1000
    pv = np.where(exact, pr - 1000, pr)
    med = float(np.median(pv))
    print(f"[probes] k={k}: median {med}, mean {pv.mean():.2f}, p99 {np.percentile(pv, 99)}, "
          f"exact-descent rows {int(exact.sum())}")
    assert med <= 10, med
    assert exact.mean() < 0.01


@pytest.mark.parametrize("shift", [-10.0, 0.0, 10.0])
@pytest.mark.parametrize("k", [8, 32, 96, 128])
def test_topk_threshold_sign(shift, k):
    """The extraction finish compares positive candidates as raw bits and falls back to order-preserving keys when
    a candidate or bound is negative (topk_row.cuh): thresholds below zero (shift -10, or k = 128 of 256 near 0),
    above zero (shift +10) and mixed, with a row-to-row spread so the warm start misses by several values."""
    n, h = 3001, 256
    rng = np.random.default_rng(k)
    x = synth.normal_f32((n, h), seed=900 + k) * rng.uniform(0.5, 2.0, size=(n, 1)).astype(np.float32)
    x = (x + np.float32(shift) + rng.normal(0, 0.3, size=(n, 1)).astype(np.float32)).astype(np.float32)
    d, i = gpu_topk(x, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri)
    assert np.array_equal(d.view(np.uint32), rd.view(np.uint32))


def test_topk_all_equal_and_signed_zero_rows():
    x = np.zeros((64, 256), np.float32)
    x[0::2] = -0.0
    x[1::4] = 0.7
    x[3::8, ::3] = -0.0
    for k in (1, 8, 32, 255, 256):
        d, i = gpu_topk(x, k)
        rd, ri = oracle.topk_cbsr(x, k)
        assert np.array_equal(i, ri) and np.array_equal(d.view(np.uint32), rd.view(np.uint32))


def test_topk_golden_example():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")))
    X = np.array([[np.float32(float(v)) for v in row] for row in g["X"]], np.float32)
    d, i = gpu_topk(X, g["k"])
    assert i.tolist() == g["idx"]
    assert np.signbit(d[3, 0])


def test_topk_strided_rows():
    x = synth.normal_f32((500, 300), 7)
    xt = _cuda(x)[:, :256]  # ld = 300 (not 16B-aligned rows): scalar path
    d, i = maxk.maxk_topk_cbsr(xt, 32)
    rd, ri = oracle.topk_cbsr(np.ascontiguousarray(x[:, :256]), 32)
    assert np.array_equal(i.cpu().numpy().astype(np.int32), ri)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), rd.view(np.uint32))


# ------------------------------------------------------------------------------------------------
# forward / backward on small graphs: ragged degrees, empty rows, duplicates, hubs split into chunks
# ------------------------------------------------------------------------------------------------
def _graph_with_hubs(n_rows, n_cols, seed, hub_deg=3000, dup=False):
    g = synth.random_csr(n_rows, n_cols, avg_deg=9.0, seed=seed, duplicates=dup)
    rng = np.random.default_rng(seed + 1)
    deg = np.diff(g.row_ptr)
    rows = []
    for i in range(n_rows):
        c = g.col_idx[g.row_ptr[i]:g.row_ptr[i + 1]]
        v = g.val[g.row_ptr[i]:g.row_ptr[i + 1]]
        if i in (1, n_rows // 2):  # two hub rows longer than any chunk (>= 256 edges)
            c = np.sort(rng.integers(0, n_cols, size=hub_deg)).astype(np.int32)
            v = rng.standard_normal(hub_deg).astype(np.float32)
        rows.append((c, v))
    deg = np.array([r[0].size for r in rows], np.int64)
    rp = np.zeros(n_rows + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = np.concatenate([r[0] for r in rows]).astype(np.int32)
    val = np.concatenate([r[1] for r in rows]).astype(np.float32)
    return synth.Csr(rp, col, val, n_cols)


def run_gpu(g, x, dy, k, use_plan=True):
    agg = MaxkAggregation(_cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val), g.n_cols, x.shape[1], k, use_plan=use_plan)
    agg.topk(_cuda(x))
    y = agg.forward().cpu().numpy()
    dxs = agg.backward(_cuda(dy)).cpu().numpy()
    d = agg.sp_data.cpu().numpy()
    i = agg.sp_idx.cpu().numpy().astype(np.int32)
    info = agg.plan.info() if agg.plan is not None else None
    agg.close()
    return d, i, y, dxs, info


# includes the paper's k sweep {2,4,8,16,32,64,96,128,192} at H=256
AGG_CASES = [(h, k) for h, k in [(64, 8), (256, 32), (256, 8), (256, 16), (256, 64), (256, 1), (256, 3), (256, 24),
                                 (256, 100), (256, 256), (128, 128), (384, 48), (100, 10), (32, 32), (512, 200),
                                 (256, 2), (256, 4), (256, 96), (256, 128), (256, 192),
                                 (1024, 64), (1024, 1024), (768, 96)]]


# Both forward layouts on every small case: spgemm_fwd_kernel with NC = EPI interleaved row buffers
# (MAXK_FWD_REP=0) and with NC = 16 replicated buffers (=2, forced: the default policy only picks it for k >= 32
# on high-degree graphs).
FWD_PATHS = pytest.mark.parametrize("fwd_path", ["0", "2"], ids=["fwd_int", "fwd_rep"])


@FWD_PATHS
@pytest.mark.parametrize("h,k", AGG_CASES)
@pytest.mark.parametrize("use_plan", [True, False])
def test_fwd_bwd_parity_small(h, k, use_plan, fwd_path, monkeypatch):
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    n_rows, n_cols = 700, 900
    g = _graph_with_hubs(n_rows, n_cols, seed=h + k, dup=(k % 2 == 1))
    x = synth.normal_f32((n_cols, h), seed=h * 7 + k)
    dy = synth.normal_f32((n_rows, h), seed=h * 11 + k)
    d, i, y, dxs, info = run_gpu(g, x, dy, k, use_plan)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri) and np.array_equal(d.view(np.uint32), rd.view(np.uint32))
    assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")
    if use_plan:
        assert info["n_split_rows"] >= 2  # the hub rows were chunked


@FWD_PATHS
@pytest.mark.parametrize("k", [8, 16, 32, 64, 96, 128, 256])
def test_fwd_bwd_parity_degree_sweep(k, fwd_path, monkeypatch):
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    """Rows of every degree 0..320 (every tail length of the long-unit chunk pipeline, both sides of the grouped
    short-row threshold), with duplicates and negative weights, h = 256."""
    h, n_cols = 256, 1200
    rng = np.random.default_rng(k)
    degs = np.concatenate([np.arange(321), rng.integers(0, 321, size=200)])
    rng.shuffle(degs)
    row_ptr = np.zeros(degs.size + 1, np.int64)
    np.cumsum(degs, out=row_ptr[1:])
    col = rng.integers(0, n_cols, size=int(row_ptr[-1])).astype(np.int32)
    val = rng.standard_normal(col.size).astype(np.float32)
    x = synth.normal_f32((n_cols, h), seed=k + 17)
    dy = synth.normal_f32((degs.size, h), seed=k + 18)
    g = synth.Csr(row_ptr, col, val, n_cols)
    d, i, y, dxs, _ = run_gpu(g, x, dy, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri)
    assert_rows_close(y, oracle.spgemm_fwd(row_ptr, col, val, rd, ri, h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(row_ptr, col, val, dy, ri), what="dXs")


@FWD_PATHS
@pytest.mark.parametrize("k", [8, 16, 32, 64])
@pytest.mark.parametrize("weights", ["mean", "one", "mixed"])
def test_uniform_weight_batches(k, weights, fwd_path, monkeypatch):
    """Batches whose edge weights are all equal skip the per-step weight broadcast (aggregate_fwd.cu /
    aggregate_bwd.cu): SAGE-mean rows (1/deg), sum rows (1), and rows where only some 32-edge batches are uniform."""
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    h = 256
    g = _graph_with_hubs(700, 900, seed=k + 5)
    deg = np.diff(g.row_ptr)
    val = np.repeat((1.0 / np.maximum(deg, 1)).astype(np.float32), deg)
    if weights == "one":
        val = np.ones_like(val)
    elif weights == "mixed":  # every other 32-edge block of each row perturbed
        pos = np.arange(val.size) - np.repeat(g.row_ptr[:-1], deg)
        val = np.where((pos // 32) % 2 == 1, val * np.float32(1.5), val).astype(np.float32)
        val[::97] = -val[::97]
    g = synth.Csr(g.row_ptr, g.col_idx, val, g.n_cols)
    x = synth.normal_f32((900, h), k + 6)
    dy = synth.normal_f32((700, h), k + 7)
    d, i, y, dxs, _ = run_gpu(g, x, dy, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")


@pytest.mark.parametrize("n_ctrs", [2, 3, 7, 32])
def test_interleaved_ticket_counters(n_ctrs, monkeypatch):
    # force the multi-counter scheduler with work stealing (normally n_ctrs = n_tix / 8192) on a small graph
    # with hub chunks, long rows and grouped short rows: every unit is processed exactly once
    monkeypatch.setenv("MAXK_SCHED_CTRS", str(n_ctrs))
    h, k = 256, 32
    g = _graph_with_hubs(700, 900, seed=41)
    x = synth.normal_f32((900, h), 8)
    dy = synth.normal_f32((700, h), 9)
    for _ in range(2):  # the counters must be reset by the last warp of each launch
        d, i, y, dxs, info = run_gpu(g, x, dy, k)
        rd, ri = oracle.topk_cbsr(x, k)
        assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")
        assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")


@pytest.mark.parametrize("h,k", [(4096, 64), (4096, 1024), (2048, 256)])
def test_max_width_aggregation(h, k):
    # the aggregation kernels' width limit (h <= 4096: the shared-memory row buffer); top-k is limited to
    # h <= 1024, so the CBSR comes from the oracle (uint16 indices)
    n_rows, n_cols = 300, 250
    g = _graph_with_hubs(n_rows, n_cols, seed=h + k, hub_deg=700)
    x = synth.normal_f32((n_cols, h), 3)
    dy = synth.normal_f32((n_rows, h), 4)
    rd, ri = oracle.topk_cbsr(x, k)
    rp_d, ci_d, va_d = _cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val)
    sd, si = _cuda(rd), _cuda(ri.astype(np.uint16))
    nnz = int(g.row_ptr[-1])
    for plan in (maxk.maxk_plan_create(rp_d, h, k), None):
        y = maxk.maxk_spgemm_fwd(rp_d, ci_d, va_d, n_cols, nnz, sd, si, h, plan=plan).cpu().numpy()
        dxs = maxk.maxk_sspmm_bwd(rp_d, ci_d, va_d, n_cols, nnz, _cuda(dy), si, plan=plan).cpu().numpy()
        assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y")
        assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")


@FWD_PATHS
@pytest.mark.parametrize("h,k", [(256, 32), (256, 8), (256, 3), (384, 48), (100, 10)])
@pytest.mark.parametrize("use_plan", [True, False])
def test_accumulating_forms(h, k, use_plan, fwd_path, monkeypatch):
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    # maxk_spgemm_fwd_acc / maxk_sspmm_bwd_acc add to the existing output (f2 overlap), hub chunks included;
    # maxk_add_f32 is an elementwise add
    n_rows, n_cols = 700, 900
    g = _graph_with_hubs(n_rows, n_cols, seed=h * 3 + k)
    x = synth.normal_f32((n_cols, h), 12)
    dy = synth.normal_f32((n_rows, h), 13)
    y0 = synth.normal_f32((n_rows, h), 14)
    d0 = synth.normal_f32((n_cols, k), 15)
    rp_d, ci_d, va_d = _cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val)
    nnz = int(g.row_ptr[-1])
    sd, si = maxk.maxk_topk_cbsr(_cuda(x), k)
    plan = maxk.maxk_plan_create(rp_d, h, k) if use_plan else None
    y = _cuda(y0)
    maxk.maxk_spgemm_fwd(rp_d, ci_d, va_d, n_cols, nnz, sd, si, h, y=y, plan=plan, accumulate=True)
    d = _cuda(d0)
    maxk.maxk_sspmm_bwd(rp_d, ci_d, va_d, n_cols, nnz, _cuda(dy), si, d_sp_data=d, plan=plan, accumulate=True)
    rd, ri = oracle.topk_cbsr(x, k)
    assert_rows_close(y.cpu().numpy(), y0 + oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what="Y+=")
    assert_rows_close(d.cpu().numpy(), d0 + oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs+=")
    a = _cuda(y0)
    maxk.maxk_add_f32(a, _cuda(x[:n_rows]))
    assert np.array_equal(a.cpu().numpy(), y0 + x[:n_rows])


def test_validators_detect_contract_violations():
    # debug-only checks of the input-value contract (maxk_validate_csr / maxk_validate_cbsr)
    h, k = 64, 8
    g = _graph_with_hubs(300, 200, seed=5)
    rp, ci = _cuda(g.row_ptr), _cuda(g.col_idx)
    assert maxk.maxk_validate_csr(rp, ci, 200) == (0, 0)
    assert maxk.maxk_validate_csr(rp, ci, 150)[1] == int((g.col_idx >= 150).sum())
    bad_rp = g.row_ptr.copy()
    bad_rp[5] = bad_rp[7]  # row 5 runs backwards into row 6's start
    assert maxk.maxk_validate_csr(_cuda(bad_rp), ci, 200)[0] >= 1
    _, si = maxk.maxk_topk_cbsr(_cuda(synth.normal_f32((50, h), 3)), k)
    assert maxk.maxk_validate_cbsr(si, h) == 0
    bad = si.clone()
    bad[3, 1] = bad[3, 0]  # not strictly ascending
    bad[7, k - 1] = h      # index out of range
    assert maxk.maxk_validate_cbsr(bad, h) == 2


@pytest.mark.parametrize("name,k", [("tiny", 8), ("flickr", 32)])
def test_cuda_graph_replay_matches_eager(name, k):
    # MaxkAggregation.capture_step: the captured pass replays with new inputs copied into the same buffers
    c = synth.CONFIGS[name]
    g = synth.config_graph(name)
    agg = MaxkAggregation(_cuda(g.row_ptr), _cuda(g.col_idx), _cuda(g.val), c.n, c.h, k)
    x, dy = _cuda(synth.normal_f32((c.n, c.h), 31)), _cuda(synth.normal_f32((c.n, c.h), 32))
    graph = agg.capture_step(x, dy)
    for seed in (41, 42):  # replay twice with different inputs
        xs, dys = synth.normal_f32((c.n, c.h), seed), synth.normal_f32((c.n, c.h), seed + 100)
        x.copy_(_cuda(xs))
        dy.copy_(_cuda(dys))
        graph.replay()
        torch.cuda.synchronize()
        rd, ri = oracle.topk_cbsr(xs, k)
        assert np.array_equal(agg.sp_idx.cpu().numpy().astype(np.int32), ri)
        assert_rows_close(agg.y.cpu().numpy(), oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, c.h), what="Y")
        assert_rows_close(agg.d_sp_data.cpu().numpy(), oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dys, ri),
                          what="dXs")
    agg.close()


def test_empty_graph_and_empty_rows():
    h, k = 256, 32
    g = synth.Csr(np.zeros(51, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32), 40)
    x = synth.normal_f32((40, h), 1)
    dy = synth.normal_f32((50, h), 2)
    for use_plan in (True, False):
        d, i, y, dxs, _ = run_gpu(g, x, dy, k, use_plan)
        assert np.all(y == 0) and y.shape == (50, h)
        assert np.all(dxs == 0) and dxs.shape == (40, k)


def test_row_block_with_offset_row_ptr():
    # zero-copy row block: row_ptr[0] != 0, col_idx/val indexed absolutely (maxk.h CSR layout)
    h, k = 256, 32
    g = synth.power_law_graph(3000, 60000, seed=3)
    r0, r1 = 1000, 2200
    rp = g.row_ptr[r0:r1 + 1].copy()
    x = synth.normal_f32((3000, h), 4)
    dy = synth.normal_f32((r1 - r0, h), 5)
    sd, si = maxk.maxk_topk_cbsr(_cuda(x), k)
    rp_d, ci_d, va_d = _cuda(rp), _cuda(g.col_idx), _cuda(g.val)
    nnz = int(rp[-1] - rp[0])
    plan = maxk.maxk_plan_create(rp_d, h, k)
    y = maxk.maxk_spgemm_fwd(rp_d, ci_d, va_d, 3000, nnz, sd, si, h, plan=plan).cpu().numpy()
    dxs = maxk.maxk_sspmm_bwd(rp_d, ci_d, va_d, 3000, nnz, _cuda(dy), si, plan=plan).cpu().numpy()
    rd, ri = oracle.topk_cbsr(x, k)
    sub = (rp - rp[0]).astype(np.int64)
    col = g.col_idx[rp[0]:rp[-1]]
    val = g.val[rp[0]:rp[-1]]
    assert_rows_close(y, oracle.spgemm_fwd(sub, col, val, rd, ri, h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(sub, col, val, dy, ri), what="dXs")


@FWD_PATHS
def test_forward_is_deterministic_and_plan_independent(fwd_path, monkeypatch):
    monkeypatch.setenv("MAXK_FWD_REP", fwd_path)
    h, k = 256, 32
    g = synth.power_law_graph(20000, 2_000_000, seed=9)
    x = synth.normal_f32((20000, h), 1)
    dy = synth.normal_f32((20000, h), 2)
    _, _, y1, dx1, info = run_gpu(g, x, dy, k, True)
    _, _, y2, dx2, _ = run_gpu(g, x, dy, k, True)
    assert info["n_split_rows"] > 0
    assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32))  # fixed per-row order, run to run
    _, _, y3, dx3, _ = run_gpu(g, x, dy, k, False)
    np.testing.assert_allclose(y1, y3, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(dx1, dx3, rtol=1e-5, atol=1e-5)


def test_adjointness_on_gpu_outputs():
    # <Y, dY> == sum(data * dXs)  (Eq. 3 forward/backward are a transpose pair)
    h, k = 256, 16
    g = synth.power_law_graph(5000, 200000, seed=13)
    x = synth.normal_f32((5000, h), 3)
    dy = synth.normal_f32((5000, h), 4)
    d, i, y, dxs, _ = run_gpu(g, x, dy, k)
    lhs = float((y.astype(np.float64) * dy).sum())
    rhs = float((d.astype(np.float64) * dxs).sum())
    assert abs(lhs - rhs) <= 1e-4 * (1 + abs(lhs))


# ------------------------------------------------------------------------------------------------
# BASELINE.json configs: tiny and Flickr-shaped in full; Reddit-shaped on sampled rows
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,k", [("tiny", 8), ("flickr", 16), ("flickr", 32), ("flickr", 64)])
def test_config_full(name, k):
    c = synth.CONFIGS[name]
    g = synth.config_graph(name)
    x = synth.normal_f32((c.n, c.h), synth.X_SEED)
    dy = synth.normal_f32((c.n, c.h), synth.DY_SEED)
    d, i, y, dxs, _ = run_gpu(g, x, dy, k)
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri) and np.array_equal(d.view(np.uint32), rd.view(np.uint32))
    assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, c.h), what="Y")
    assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs")


def _sample_rows(deg: np.ndarray, n_random: int, seed: int):
    rng = np.random.default_rng(seed)
    top = np.argsort(-deg, kind="stable")[:64]         # the hub rows (split into chunks)
    rnd = rng.choice(deg.size, size=n_random, replace=False)
    return np.unique(np.concatenate([top, rnd, [0, deg.size - 1]])).astype(np.int64)


@pytest.mark.slow
def test_headline_config_all_rows():
    """The metric's configuration (Reddit-shaped, k=32), in the launch configuration bench.py times (plan,
    dynamic scheduling): CBSR bit-exact on every row, Y and dXs on EVERY row against the fp64 oracle; the worst
    err/tol must stay below 0.25 (investigate above 0.25 tol before relaxing anything)."""
    c = synth.CONFIGS["reddit"]
    g = synth.config_graph("reddit")
    x = synth.normal_f32((c.n, c.h), synth.X_SEED)
    dy = synth.normal_f32((c.n, c.h), synth.DY_SEED)
    d, i, y, dxs, _ = run_gpu(g, x, dy, 32)
    rd, ri = oracle.topk_cbsr(x, 32)
    assert np.array_equal(i, ri) and np.array_equal(d.view(np.uint32), rd.view(np.uint32))
    r_y = assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, c.h), what="Y (all rows)")
    r_d = assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what="dXs (all rows)")
    assert max(r_y, r_d) < 0.25, (r_y, r_d)


@pytest.mark.slow
@pytest.mark.parametrize("name,k", [("reddit", 8), ("reddit", 16), ("reddit", 64), ("proteins", 32),
                                    ("products", 32), ("yelp", 96)])
def test_config_sampled(name, k):
    c = synth.CONFIGS[name]
    g = synth.config_graph(name)
    x = synth.normal_f32((c.n, c.h), synth.X_SEED)
    dy = synth.normal_f32((c.n, c.h), synth.DY_SEED)
    d, i, y, dxs, info = run_gpu(g, x, dy, k)
    deg = np.diff(g.row_ptr)
    rows = _sample_rows(deg, 1500, seed=k)
    # top-k: sampled rows bit-exact
    rd, ri = oracle.topk_cbsr(x[rows], k)
    assert np.array_equal(i[rows], ri) and np.array_equal(d[rows].view(np.uint32), rd.view(np.uint32))
    # forward rows need the full CBSR: the oracle's own top-k over all rows
    rd_all, ri_all = oracle.topk_cbsr(x, k)
    assert np.array_equal(i, ri_all)
    assert_rows_close(y[rows], oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd_all, ri_all, c.h, rows=rows),
                      what="Y")
    in_deg = np.bincount(g.col_idx, minlength=c.n)
    rows_b = _sample_rows(in_deg, 1500, seed=k + 1)
    assert_rows_close(dxs[rows_b], oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri_all, rows=rows_b),
                      what="dXs")


def test_width_sequence_reuses_larger_smem_limit():
    """the dynamic shared-memory limit belongs to the kernel; a call with a smaller footprint must not
    leave it lowered under a cached larger one (h = 1024 -> 512 -> 1024 at k = 32, same kernel instance)."""
    n_rows, n_cols = 300, 400
    g = _graph_with_hubs(n_rows, n_cols, seed=5, dup=False)
    for h in (1024, 512, 1024):
        x = synth.normal_f32((n_cols, h), seed=h)
        dy = synth.normal_f32((n_rows, h), seed=h + 1)
        d, i, y, dxs, _ = run_gpu(g, x, dy, 32)
        rd, ri = oracle.topk_cbsr(x, 32)
        assert np.array_equal(i, ri)
        assert_rows_close(y, oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, h), what=f"Y h={h}")
        assert_rows_close(dxs, oracle.sspmm_bwd(g.row_ptr, g.col_idx, g.val, dy, ri), what=f"dXs h={h}")


def test_launch_count_increments():
    before = maxk.launch_count()
    gpu_topk(synth.normal_f32((10, 64), 1), 4)
    assert maxk.launch_count() == before + 1


# ------------------------------------------------------------------------------------------------
# f1: MaxK backward scatter (PAPER.md:226 Def. ii) — bit-exact vs oracle densify
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("h,k", [(256, 32), (256, 8), (64, 8), (100, 7), (384, 48), (256, 256)])
def test_cbsr_scatter_bit_exact(h, k):
    n = 1000
    x = synth.normal_f32((n, h), h + k)
    g = synth.normal_f32((n, k), h * k)
    _, si = maxk.maxk_topk_cbsr(_cuda(x), k)
    dx = maxk.maxk_cbsr_scatter(_cuda(g), si, h).cpu().numpy()
    ref = oracle.densify(g, si.cpu().numpy().astype(np.int32), h)
    assert np.array_equal(dx.astype(np.float64), ref)


def test_cbsr_scatter_strided_output():
    n, h, k = 300, 256, 16
    x = synth.normal_f32((n, h), 5)
    g = synth.normal_f32((n, k), 6)
    _, si = maxk.maxk_topk_cbsr(_cuda(x), k)
    big = torch.full((n, h + 3), 7.0, device="cuda")
    maxk.maxk_cbsr_scatter(_cuda(g), si, h, dx=big[:, :h])
    out = big.cpu().numpy()
    assert np.array_equal(out[:, :h].astype(np.float64), oracle.densify(g, si.cpu().numpy().astype(np.int32), h))
    assert np.all(out[:, h:] == 7.0)  # the padding columns are not touched

