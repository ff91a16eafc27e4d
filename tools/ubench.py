"""Run the ceiling microbenchmarks (tools/ubench/ubench.cu) on the Reddit-shaped workload and compare them with
the aggregation kernels (SURVEY.md §8(d) d.6 "true-limiter evidence").

    python tools/ubench.py [--config reddit] [--k 32] [--out profiles/r01/ubench.json]

For each component of the k=32 inner loop it prints the time the component alone needs for nnz edges:
  smem_rmw     forward's shared-memory scatter (LDS+FFMA+STS of 32 random columns per edge)
  lds_gather   backward's shared-memory gather (32 random columns per edge)
  cbsr_gather  forward's global part (col/val stream + 160-B CBSR row gather from L2)
  red          backward's 128-B red.global.add.v4 per edge into the L2-resident d_sp_data
and the full kernels' times from the same process, so fwd/bwd can be read as fractions of these ceilings.
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402
from paper_2312_08656_b200.layer import MaxkAggregation  # noqa: E402

SRC = os.path.join(ROOT, "tools", "ubench", "ubench.cu")
LIB = os.path.join(ROOT, "tools", "ubench", "libubench.so")


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                               "-Xcompiler", "-fPIC", "-cudart", "static", "-o", LIB, SRC])
    lib = ctypes.CDLL(LIB)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.ubench_smem_rmw.argtypes = [vp, i32, i64, vp, i32]
    lib.ubench_lds_gather.argtypes = [vp, i32, i64, vp, i32]
    lib.ubench_cbsr_gather.argtypes = [vp, vp, i64, vp, vp, vp, i32]
    lib.ubench_red.argtypes = [vp, i64, vp, i32]
    lib.ubench_red_scalar.argtypes = [vp, i64, vp, i32, i32]
    lib.ubench_red_masked.argtypes = [vp, i64, vp, i32, i32]
    lib.ubench_red_bulk.argtypes = [vp, i64, vp, i32]
    lib.ubench_stg.argtypes = [vp, i64, vp, i32]
    for f in ("ubench_smem_rmw", "ubench_lds_gather", "ubench_cbsr_gather", "ubench_red", "ubench_red_scalar",
              "ubench_red_masked", "ubench_red_bulk", "ubench_stg"):
        getattr(lib, f).restype = ctypes.c_float
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    assert args.k == 32, "the microbenchmarks mirror the k=32 lane mapping"
    lib = build()
    cfg = synth.CONFIGS[args.config]
    g = synth.config_graph(cfg.name)
    dev = torch.device("cuda")
    x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).to(dev)
    dy = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)).to(dev)
    rp, ci, va = (torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col_idx, g.val))
    agg = MaxkAggregation(rp, ci, va, cfg.n, cfg.h, args.k)
    agg.topk(x)
    sink = torch.zeros(1, device=dev)
    red_out = torch.zeros((cfg.n, args.k), device=dev)
    nnz = g.nnz
    res = {"config": cfg.name, "k": args.k, "nnz": nnz}
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    res["smem_rmw_ms"] = lib.ubench_smem_rmw(ptr(agg.sp_idx), min(cfg.n, 4096), nnz, ptr(sink), args.reps)
    res["lds_gather_ms"] = lib.ubench_lds_gather(ptr(agg.sp_idx), min(cfg.n, 4096), nnz, ptr(sink), args.reps)
    res["cbsr_gather_ms"] = lib.ubench_cbsr_gather(ptr(ci), ptr(va), nnz, ptr(agg.sp_data), ptr(agg.sp_idx),
                                                   ptr(sink), args.reps)
    res["red_ms"] = lib.ubench_red(ptr(ci), nnz, ptr(red_out), args.reps)
    # RED variants: scalar lanes; v4 into a 1 MB / 8 MB target; TMA bulk reduce (cp.reduce.async.bulk)
    res["red_scalar_ms"] = lib.ubench_red_scalar(ptr(ci), nnz, ptr(red_out), 0x7fffffff, args.reps)
    res["red_v4_1MB_target_ms"] = lib.ubench_red_masked(ptr(ci), nnz, ptr(red_out), 8191, args.reps)
    res["red_v4_8MB_target_ms"] = lib.ubench_red_masked(ptr(ci), nnz, ptr(red_out), 65535, args.reps)
    res["red_bulk_ms"] = lib.ubench_red_bulk(ptr(ci), nnz, ptr(red_out), args.reps)
    res["stg_same_pattern_ms"] = lib.ubench_stg(ptr(ci), nnz, ptr(red_out), args.reps)
    # full kernels, same process
    for name, fn in (("fwd_ms", agg.forward), ("bwd_ms", lambda: agg.backward(dy))):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / args.reps
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    clk = 1.965e9
    for key in ("smem_rmw_ms", "lds_gather_ms", "cbsr_gather_ms", "red_ms", "fwd_ms", "bwd_ms"):
        res[key.replace("_ms", "_cycles_per_edge_per_sm")] = res[key] * 1e-3 * clk * sms / nnz
    # ceilings: the forward needs the scatter AND the gathers on the same L1tex pipe; the backward the gather,
    # the index load and the reductions
    res["fwd_vs_smem_rmw"] = res["smem_rmw_ms"] / res["fwd_ms"]
    res["fwd_vs_rmw_plus_gather"] = (res["smem_rmw_ms"] + res["cbsr_gather_ms"]) / res["fwd_ms"]
    res["bwd_vs_red"] = res["red_ms"] / res["bwd_ms"]
    res["bwd_vs_lds_plus_red"] = (res["lds_gather_ms"] + res["red_ms"]) / res["bwd_ms"]
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    agg.close()


if __name__ == "__main__":
    main()
