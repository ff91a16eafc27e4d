"""A/B: the backward SSpMM reading the column-ordered sp_idx vs the bank-balanced copy's sp_bidx (same sets; the
staged dY row's LDS gathers see fewer bank conflicts in the banked order, tools/banksim_banked.py).
usage: python tools/ab_bwd_banked.py [config] [k] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
R = int(sys.argv[3]) if len(sys.argv) > 3 else 20
c = synth.CONFIGS[name]
g = synth.config_graph(name)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (g.row_ptr, g.col_idx, g.val))
x = torch.from_numpy(synth.normal_f32((c.n, c.h), synth.X_SEED)).cuda()
dy = torch.from_numpy(synth.normal_f32((c.n, c.h), synth.DY_SEED)).cuda()
sd, si, bd, bi = maxk.maxk_topk_cbsr_banked(x, k)
plan = maxk.maxk_plan_create(rp, c.h, k)
out = torch.empty((c.n, k), device="cuda")


def t(idx):
    for _ in range(3):
        maxk.maxk_sspmm_bwd(rp, ci, va, c.n, g.nnz, dy, idx, d_sp_data=out, plan=plan)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        maxk.maxk_sspmm_bwd(rp, ci, va, c.n, g.nnz, dy, idx, d_sp_data=out, plan=plan)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R


for rnd in range(2):
    print(f"{name} k={k} bwd column-order {t(si):.3f} ms  banked {t(bi):.3f} ms")
