"""Small end-to-end runs of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--flickr]
Covers: top-k (fast, vector and strided paths, uint8/uint16, probe statistics, the pair and bank-balanced copies),
forward (both row-buffer layouts, NC = EPI and NC = 16, from the two-block, pair and bank-balanced CBSR) and backward vector kernels (k=8,16,32,64,128),
generic kernels (k=3, 24, 100), plan and plan-free scheduling, hub rows split into chunks, empty rows,
n_cols != n_rows. Exits non-zero on a parity failure against the CPU oracle.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402


def run(n_rows, n_cols, h, k, use_plan, seed):
    g = synth.random_csr(n_rows, n_cols, avg_deg=6.0, seed=seed)
    # one hub row longer than the minimum chunk (256) so the plan splits it
    rng = np.random.default_rng(seed)
    deg = np.diff(g.row_ptr)
    hub = np.sort(rng.integers(0, n_cols, size=600)).astype(np.int32)
    cols = [hub if i == 1 else g.col_idx[g.row_ptr[i]:g.row_ptr[i + 1]] for i in range(n_rows)]
    vals = [rng.standard_normal(600).astype(np.float32) if i == 1 else g.val[g.row_ptr[i]:g.row_ptr[i + 1]]
            for i in range(n_rows)]
    deg = np.array([c.size for c in cols])
    rp = np.zeros(n_rows + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = np.concatenate(cols).astype(np.int32)
    val = np.concatenate(vals).astype(np.float32)
    x = synth.normal_f32((n_cols, h), seed)
    dy = synth.normal_f32((n_rows, h), seed + 1)
    dev = torch.device("cuda")
    rp_d, ci_d, va_d = (torch.from_numpy(a).to(dev) for a in (rp, col, val))
    sd, si = maxk.maxk_topk_cbsr(torch.from_numpy(x).to(dev), k)
    plan = maxk.maxk_plan_create(rp_d, h, k) if use_plan else None
    y = maxk.maxk_spgemm_fwd(rp_d, ci_d, va_d, n_cols, int(rp[-1]), sd, si, h, plan=plan)
    d = maxk.maxk_sspmm_bwd(rp_d, ci_d, va_d, n_cols, int(rp[-1]), torch.from_numpy(dy).to(dev), si, plan=plan)
    torch.cuda.synchronize()
    rd, ri = oracle.topk_cbsr(x, k)
    assert np.array_equal(si.cpu().numpy().astype(np.int32), ri)
    yr = oracle.spgemm_fwd(rp, col, val, rd, ri, h)
    dr = oracle.sspmm_bwd(rp, col, val, dy, ri)
    for got, ref in ((y.cpu().numpy(), yr), (d.cpu().numpy(), dr)):
        err = np.abs(got - ref).max(axis=1)
        assert np.all(err <= 1e-5 * (1 + np.abs(ref).max(axis=1))), (h, k, use_plan)
    if maxk.pairs_supported(h, k):  # the CBSR pair layout (k in {8, 16}, always the interleaved row buffers)
        _, _, sp = maxk.maxk_topk_cbsr_pairs(torch.from_numpy(x).to(dev), k)
        yp = maxk.maxk_spgemm_fwd_pairs(rp_d, ci_d, va_d, n_cols, int(rp[-1]), sp, h, plan=plan)
        torch.cuda.synchronize()
        if os.environ.get("MAXK_FWD_REP") == "0":  # the same interleaved layout: bit-identical
            assert torch.equal(yp, y), (h, k, use_plan)
        err = np.abs(yp.cpu().numpy() - yr).max(axis=1)
        assert np.all(err <= 1e-5 * (1 + np.abs(yr).max(axis=1))), (h, k, use_plan, "pairs")
    if maxk.banked_supported(h, k):  # the bank-balanced copy (k in {32, 64, 128}) read by the forward
        _, _, bd, bi = maxk.maxk_topk_cbsr_banked(torch.from_numpy(x).to(dev), k)
        yb = maxk.maxk_spgemm_fwd(rp_d, ci_d, va_d, n_cols, int(rp[-1]), bd, bi, h, plan=plan)
        torch.cuda.synchronize()
        err = np.abs(yb.cpu().numpy() - yr).max(axis=1)
        assert np.all(err <= 1e-5 * (1 + np.abs(yr).max(axis=1))), (h, k, use_plan, "banked")
    dx = maxk.maxk_cbsr_scatter(d, si, h)  # d_sp_data and sp_idx are both [n_cols x k]
    assert np.array_equal(dx.cpu().numpy().astype(np.float64), oracle.densify(d.cpu().numpy(), ri, h))
    if plan is not None:
        plan.close()


def flickr():
    """One layer pass on the Flickr-shaped config (SURVEY §4 layer 4) through the product path, checked on sampled
    rows against the oracle."""
    from paper_2312_08656_b200.layer import MaxkAggregation
    c = synth.CONFIGS["flickr"]
    g = synth.config_graph("flickr")
    dev = torch.device("cuda")
    x = synth.normal_f32((c.n, c.h), synth.X_SEED)
    dy = synth.normal_f32((c.n, c.h), synth.DY_SEED)
    agg = MaxkAggregation(*(torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col_idx, g.val)), c.n, c.h, 32)
    y, d = agg.step(torch.from_numpy(x).to(dev), torch.from_numpy(dy).to(dev))
    torch.cuda.synchronize()
    rows = np.arange(0, c.n, 97, dtype=np.int64)
    rd, ri = oracle.topk_cbsr(x, 32)
    yr = oracle.spgemm_fwd(g.row_ptr, g.col_idx, g.val, rd, ri, c.h, rows=rows)
    assert np.all(np.abs(y.cpu().numpy()[rows] - yr).max(axis=1) <= 1e-5 * (1 + np.abs(yr).max(axis=1)))
    agg.close()
    print("sanitize_run flickr ok")


def main():
    cases = [(256, 32), (256, 8), (256, 16), (256, 64), (256, 128), (256, 3), (256, 24), (256, 100), (64, 8),
             (384, 48), (100, 10)]
    for mode in ("0", "2"):  # both forward layouts: NC = EPI interleaved and NC = 16 replicated (forced)
        os.environ["MAXK_FWD_REP"] = mode
        for i, (h, k) in enumerate(cases):
            for use_plan in (True, False):
                run(150, 170, h, k, use_plan, seed=i)
    del os.environ["MAXK_FWD_REP"]
    # interleaved ticket counters with work stealing (normally only on large graphs)
    os.environ["MAXK_SCHED_CTRS"] = "3"
    for i, (h, k) in enumerate([(256, 32), (256, 8), (256, 128)]):
        run(150, 170, h, k, True, seed=100 + i)
    del os.environ["MAXK_SCHED_CTRS"]
    # accumulating forms (f2), the add kernel and the debug validators
    g = synth.random_csr(150, 170, avg_deg=6.0, seed=7)
    dev = torch.device("cuda")
    rp_d, ci_d, va_d = (torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col_idx, g.val))
    x = synth.normal_f32((170, 256), 8)
    dy = synth.normal_f32((150, 256), 9)
    sd, si = maxk.maxk_topk_cbsr(torch.from_numpy(x).to(dev), 32)
    plan = maxk.maxk_plan_create(rp_d, 256, 32)
    y = torch.zeros((150, 256), device=dev)
    maxk.maxk_spgemm_fwd(rp_d, ci_d, va_d, 170, g.nnz, sd, si, 256, y=y, plan=plan, accumulate=True)
    d = torch.zeros((170, 32), device=dev)
    maxk.maxk_sspmm_bwd(rp_d, ci_d, va_d, 170, g.nnz, torch.from_numpy(dy).to(dev), si, d_sp_data=d, plan=plan,
                        accumulate=True)
    maxk.maxk_add_f32(d, d.clone())
    assert maxk.maxk_validate_csr(rp_d, ci_d, 170) == (0, 0) and maxk.maxk_validate_cbsr(si, 256) == 0
    torch.cuda.synchronize()
    plan.close()
    # fused Eq. 1 kernel (tcgen05 + TMA + TMEM + the staged warp-per-row epilogue): a ragged tile tail, and more
    # tiles than CTAs (both TMEM accumulator stages and the mbarrier phases of several tiles per CTA)
    g = torch.Generator().manual_seed(3)
    for n_rows, f_in, h, k in ((300, 128, 256, 32), (20000, 64, 128, 8)):
        x = torch.randn((n_rows, f_in), generator=g).to(torch.bfloat16).cuda()
        w = (torch.randn((h, f_in), generator=g) / 8).to(torch.bfloat16).cuda()
        z = torch.empty((n_rows, h), device="cuda")
        sd, si = maxk.maxk_linear_topk_cbsr(x, w, k, z_out=z)
        torch.cuda.synchronize()
        rd, ri = oracle.topk_cbsr(z.cpu().numpy(), k)
        assert np.array_equal(si.cpu().numpy().astype(np.int32), ri)
    _, _, probes = maxk.maxk_topk_cbsr_probe_stats(torch.from_numpy(synth.normal_f32((300, 256), 5)).cuda(), 32)
    torch.cuda.synchronize()
    print("sanitize_run ok:", len(cases) * 4 + 6, "cases")


if __name__ == "__main__":
    flickr() if "--flickr" in sys.argv else main()
