"""Device time of maxk_topk_cbsr alone on a config's X (quick A/B; not the driver's bench line).
usage: python tools/time_topk.py [config] [k] ...   (MAXK_TOPK_PATH=probe selects the probe kernel)"""
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
    d = torch.empty((cfg.n, k), device="cuda")
    i = torch.empty((cfg.n, k), device="cuda", dtype=maxk.idx_dtype(cfg.h))
    for _ in range(5):
        maxk.maxk_topk_cbsr(x, k, d, i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    R = 50
    for _ in range(R):
        maxk.maxk_topk_cbsr(x, k, d, i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    by = cfg.n * cfg.h * 4 + cfg.n * k * (4 + (1 if cfg.h <= 256 else 2))
    print(f"{name} k={k} path={os.environ.get('MAXK_TOPK_PATH', 'default')} {ms:.4f} ms {by / ms / 1e6:.0f} GB/s")
