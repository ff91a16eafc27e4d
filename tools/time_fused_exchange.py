"""Device time of the fused-exchange kernels against their plain forms, on ONE GPU.

One rank's share of the Reddit-shaped layer at G ranks (its nnz-balanced row block, columns remapped to slots):
  topk        maxk_topk_cbsr into the rank's block of its replica            vs  maxk_topk_cbsr_multi into all G
  bwd         maxk_sspmm_bwd into an Nc x k partial (then a reduce-scatter)  vs  maxk_sspmm_bwd_owners into the G
              owners' R_max x k blocks
On one GPU the "peer" replicas and blocks are this device's memory, so this measures the kernels' own cost of the
fusion (G stores per row, owner routing per edge), not NVLink.
usage: python tools/time_fused_exchange.py [config] [k] [G]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402
from paper_2312_08656_b200.partition import partition_rows_by_nnz, remap_columns  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    G = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    c = synth.CONFIGS[name]
    full = synth.config_graph(name)
    part = partition_rows_by_nnz(full.row_ptr, G)
    R, Nc = part.r_max, part.n_slots
    r0, r1 = part.rows(0)
    blk = synth.config_graph(name, rows=(r0, r1))
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (blk.row_ptr, remap_columns(blk.col_idx, part), blk.val))
    nnz = int(blk.row_ptr[-1])
    x = torch.from_numpy(synth.normal_f32((r1 - r0, c.h), synth.X_SEED, row_offset=r0)).cuda()
    dy = torch.from_numpy(synth.normal_f32((r1 - r0, c.h), synth.DY_SEED, row_offset=r0)).cuda()
    n = r1 - r0
    sd = [torch.zeros((Nc, k), device="cuda") for _ in range(G)]
    si = [torch.zeros((Nc, k), dtype=torch.uint8, device="cuda") for _ in range(G)]
    # fill every replica with the full mask (as after an exchange): each block from its own rows' top-k
    for g in range(G):
        a, b = part.rows(g)
        xg = torch.from_numpy(synth.normal_f32((b - a, c.h), synth.X_SEED, row_offset=a)).cuda()
        maxk.maxk_topk_cbsr_multi(xg, k, [t[g * R:g * R + b - a] for t in sd], [t[g * R:g * R + b - a] for t in si])
    plan = maxk.maxk_plan_create(rp, c.h, k)
    dpart = torch.empty((Nc, k), device="cuda")
    blocks = [torch.zeros((R, k), device="cuda") for _ in range(G)]
    ptrs = torch.tensor([t.data_ptr() for t in blocks], dtype=torch.int64, device="cuda")
    res = {"config": name, "k": k, "G": G, "rank_rows": n, "rank_nnz": nnz,
           "topk_ms": timed(lambda: maxk.maxk_topk_cbsr(x, k, sd[0][:n], si[0][:n])),
           "topk_multi_ms": timed(lambda: maxk.maxk_topk_cbsr_multi(x, k, [t[:n] for t in sd], [t[:n] for t in si])),
           "bwd_partial_ms": timed(lambda: maxk.maxk_sspmm_bwd(rp, ci, va, Nc, nnz, dy, si[0], d_sp_data=dpart,
                                                               plan=plan)),
           "bwd_owners_ms": timed(lambda: maxk.maxk_sspmm_bwd_owners(rp, ci, va, Nc, nnz, dy, si[0], R, ptrs,
                                                                     plan=plan)),
           "note": "one GPU: the G destinations are this device's memory (kernel cost of the fusion, not NVLink)"}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
