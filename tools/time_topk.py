"""Device time of maxk_topk_cbsr alone on a config's X, every kernel path A/B in one process (not the driver's
bench line). Outputs of each path are compared bit-exactly with the default path; the probe statistic of the
default kernel (maxk_topk_cbsr_probe_stats) is summarised.
usage: python tools/time_topk.py [config k] ...   (paths: default, newton, probe via MAXK_TOPK_PATH)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402

args = sys.argv[1:] or ["reddit", "32", "products", "32"]
for name, k in zip(args[::2], args[1::2]):
    k = int(k)
    cfg = synth.CONFIGS[name]
    x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).cuda()
    by = cfg.n * cfg.h * 4 + cfg.n * k * (4 + (1 if cfg.h <= 256 else 2))
    res = {"config": name, "k": k}
    ref = None
    for path in ("default", "newton", "probe"):
        if path == "default":
            os.environ.pop("MAXK_TOPK_PATH", None)
        else:
            os.environ["MAXK_TOPK_PATH"] = path
        d = torch.empty((cfg.n, k), device="cuda")
        i = torch.empty((cfg.n, k), device="cuda", dtype=maxk.idx_dtype(cfg.h))
        for _ in range(5):
            maxk.maxk_topk_cbsr(x, k, d, i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        R = 50
        e0.record()
        for _ in range(R):
            maxk.maxk_topk_cbsr(x, k, d, i)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / R
        same = None
        if ref is None:
            ref = (d.clone(), i.clone())
        else:
            same = bool(torch.equal(i, ref[1]) and torch.equal(d.view(torch.int32), ref[0].view(torch.int32)))
        res[path] = {"ms": round(ms, 4), "GBps": round(by / ms / 1e6), "same_as_default": same}
    os.environ.pop("MAXK_TOPK_PATH", None)
    try:
        _, _, pr = maxk.maxk_topk_cbsr_probe_stats(x, k)
        pr = pr.cpu()
        exact = pr >= 1000
        pv = pr.clone()
        pv[exact] -= 1000
        res["probes"] = {"median": float(pv.float().median()), "mean": float(pv.float().mean()),
                         "p99": float(pv.float().quantile(0.99)) if pv.numel() < 16_000_000 else None,
                         "max": int(pv.max()), "exact_descent_rows": int(exact.sum())}
    except Exception as e:  # path without statistics
        res["probes"] = str(e)
    print(json.dumps(res), flush=True)
