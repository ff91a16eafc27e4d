"""Run the backward SSpMM R times on a config (for ncu captures of one kernel; not a bench line).
usage: python tools/run_bwd.py CONFIG K N_BLOCKS [R]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402

name, k, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
R = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = synth.CONFIGS[name]
g = synth.config_graph(name)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (g.row_ptr, g.col_idx, g.val))
x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).cuda()
dy = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)).cuda()
sd, si = maxk.maxk_topk_cbsr(x, k)
plan = maxk.maxk_plan_create(rp, cfg.h, k)
print("blocks", maxk.maxk_plan_set_column_blocks(plan, rp, ci, cfg.n, k, 1, n_blocks=nb))
out = torch.empty((cfg.n, k), device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    maxk.maxk_sspmm_bwd(rp, ci, va, cfg.n, g.nnz, dy, si, d_sp_data=out, plan=plan)
e1.record()
torch.cuda.synchronize()
print("ms per bwd", e0.elapsed_time(e1) / R)
