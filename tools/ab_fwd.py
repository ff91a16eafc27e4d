"""A/B of forward SpGEMM variants selected by environment knobs (not a bench line).
usage: python tools/ab_fwd.py CONFIG:K [CONFIG:K ...] [--modes 'MAXK_FWD_REP=0;MAXK_FWD_REP=1' ] [--reps R]
Times each mode on the same inputs (CUDA events, mean of R launches after warm-up) and reports the max
row-relative difference of Y against the first mode."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cases", nargs="+")
ap.add_argument("--modes", default="MAXK_FWD_REP=0;MAXK_FWD_REP=1")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--stage", default="fwd", choices=["fwd", "bwd"])
args = ap.parse_args()
modes = [m for m in args.modes.split(";")]


def set_mode(m):
    for kv in m.split(","):
        if kv:
            k, v = kv.split("=")
            os.environ[k] = v


def clear_mode(m):
    for kv in m.split(","):
        if kv:
            os.environ.pop(kv.split("=")[0], None)


for case in args.cases:
    name, k = case.split(":")
    k = int(k)
    cfg = synth.CONFIGS[name]
    g = synth.config_graph(name)
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (g.row_ptr, g.col_idx, g.val))
    x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).cuda()
    dy = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)).cuda()
    sd, si = maxk.maxk_topk_cbsr(x, k)
    plan = maxk.maxk_plan_create(rp, cfg.h, k)
    y = torch.empty((cfg.n, cfg.h), device="cuda")
    out = torch.empty((cfg.n, k), device="cuda")
    ref = None
    res = {"case": case}
    for m in modes:
        set_mode(m)

        def run():
            if args.stage == "fwd":
                maxk.maxk_spgemm_fwd(rp, ci, va, cfg.n, g.nnz, sd, si, cfg.h, y=y, plan=plan)
            else:
                maxk.maxk_sspmm_bwd(rp, ci, va, cfg.n, g.nnz, dy, si, d_sp_data=out, plan=plan)

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / args.reps
        o = (y if args.stage == "fwd" else out).clone()
        if ref is None:
            ref = o
            diff = 0.0
        else:
            diff = ((o - ref).abs().amax(1) / (1 + ref.abs().amax(1))).max().item()
        res[m] = {"ms": round(t, 4), "max_row_rel_diff": diff}
        clear_mode(m)
    print(json.dumps(res), flush=True)
