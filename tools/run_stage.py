"""Run one hot-path stage R times on a config (for ncu captures of one kernel; not a bench line).
usage: python tools/run_stage.py CONFIG K STAGE [R]     STAGE in {topk, fwd, bwd}"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402

name, k, stage = sys.argv[1], int(sys.argv[2]), sys.argv[3]
R = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = synth.CONFIGS[name]
g = synth.config_graph(name)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (g.row_ptr, g.col_idx, g.val))
x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).cuda()
dy = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)).cuda()
sd, si = maxk.maxk_topk_cbsr(x, k)
plan = maxk.maxk_plan_create(rp, cfg.h, k)
y = torch.empty((cfg.n, cfg.h), device="cuda")
out = torch.empty((cfg.n, k), device="cuda")


# the layer path's layouts (layer.MaxkAggregation / dist.CudaOps): the CBSR pair layout where it exists (k in {8, 16})
pb = maxk.banked_default(cfg.h, k, cfg.n, g.nnz)
pairs = maxk.maxk_topk_cbsr_pairs(x, k, sd, si, banked=pb)[2] if maxk.pairs_default(cfg.h, k) else None
# ... and the bank-balanced copy where it exists (k in {32, 64, 128})
banked = maxk.maxk_topk_cbsr_banked(x, k, sd, si)[2:] if pb and pairs is None else None


def run():
    if stage == "topk":
        if pairs is not None:
            maxk.maxk_topk_cbsr_pairs(x, k, sd, si, pairs, banked=pb)
        elif banked is not None:
            maxk.maxk_topk_cbsr_banked(x, k, sd, si, *banked)
        else:
            maxk.maxk_topk_cbsr(x, k, sd, si)
    elif stage == "fwd":
        if pairs is not None:
            maxk.maxk_spgemm_fwd_pairs(rp, ci, va, cfg.n, g.nnz, pairs, cfg.h, y=y, plan=plan)
        else:
            bd, bi = banked if banked is not None else (sd, si)
            maxk.maxk_spgemm_fwd(rp, ci, va, cfg.n, g.nnz, bd, bi, cfg.h, y=y, plan=plan)
    else:
        maxk.maxk_sspmm_bwd(rp, ci, va, cfg.n, g.nnz, dy, si, d_sp_data=out, plan=plan)


run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    run()
e1.record()
torch.cuda.synchronize()
print(stage, "ms", e0.elapsed_time(e1) / R)
