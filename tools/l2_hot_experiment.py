"""Experiment (not the product): how much do products-shaped forward/backward gain if the hot CBSR rows (highest
in-degree columns) stay in L2?  Relabels the graph's columns by in-degree (hot rows first, contiguous) and times
maxk_spgemm_fwd / maxk_sspmm_bwd (a) on the original labels, (b) relabelled, (c) relabelled with a persisting-L2
access-policy window over the hot prefix of sp_data / sp_idx / d_sp_data.
usage: python tools/l2_hot_experiment.py [config] [hot_fraction]"""
import os
import sys

import numpy as np
import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "products"
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
k = 32
cfg = synth.CONFIGS[name]
g = synth.config_graph(name)
indeg = np.bincount(g.col_idx, minlength=cfg.n)
order = np.argsort(-indeg, kind="stable")
new_id = np.empty(cfg.n, np.int32)
new_id[order] = np.arange(cfg.n, dtype=np.int32)
hot = int(frac * cfg.n)
print(f"{name}: top {frac:.0%} of columns ({hot} rows) receive {indeg[order[:hot]].sum() / indeg.sum():.1%} of gathers")
dev = torch.device("cuda")
rp = torch.from_numpy(g.row_ptr).to(dev)
va = torch.from_numpy(g.val).to(dev)
cols = {"original": torch.from_numpy(g.col_idx).to(dev), "relabelled": torch.from_numpy(new_id[g.col_idx]).to(dev)}
x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).to(dev)
dy = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)).to(dev)
sd, si = maxk.maxk_topk_cbsr(x, k)
plan = maxk.maxk_plan_create(rp, cfg.h, k)
y = torch.empty((cfg.n, cfg.h), device=dev)
dsd = torch.empty((cfg.n, k), device=dev)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def window(ptr, nbytes, on=True):
    st = torch.cuda.current_stream().cuda_stream
    attr = rt.cudaStreamAttrValue()
    w = attr.accessPolicyWindow
    w.base_ptr = ptr if on else 0
    w.num_bytes = nbytes if on else 0
    w.hitRatio = 1.0
    w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    attr.accessPolicyWindow = w
    err, = rt.cudaStreamSetAttribute(st, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, attr)
    assert err == rt.cudaError_t.cudaSuccess, err


err, mx = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err2, l2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, mx)
print("L2", l2, "max persisting", mx, "set:", err)
for label, ci in cols.items():
    f = lambda: maxk.maxk_spgemm_fwd(rp, ci, va, cfg.n, g.nnz, sd, si, cfg.h, y=y, plan=plan)  # noqa: E731
    b = lambda: maxk.maxk_sspmm_bwd(rp, ci, va, cfg.n, g.nnz, dy, si, d_sp_data=dsd, plan=plan)  # noqa: E731
    print(f"{label:10s} fwd {timed(f):.3f} ms  bwd {timed(b):.3f} ms")
ci = cols["relabelled"]
for nbytes_rows in (hot, hot // 2):
    window(sd.data_ptr(), nbytes_rows * k * 4)
    tf = timed(lambda: maxk.maxk_spgemm_fwd(rp, ci, va, cfg.n, g.nnz, sd, si, cfg.h, y=y, plan=plan))
    window(dsd.data_ptr(), nbytes_rows * k * 4)
    tb = timed(lambda: maxk.maxk_sspmm_bwd(rp, ci, va, cfg.n, g.nnz, dy, si, d_sp_data=dsd, plan=plan))
    window(0, 0, on=False)
    rt.cudaCtxResetPersistingL2Cache()
    print(f"relabelled + persisting window over {nbytes_rows} hot rows ({nbytes_rows * k * 4 / 1e6:.0f} MB data): "
          f"fwd {tf:.3f} ms  bwd {tb:.3f} ms")
