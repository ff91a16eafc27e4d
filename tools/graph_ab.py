"""Eager launches vs CUDA-graph replay of one layer pass (top-k -> fwd -> bwd) on a config (A/B, not a bench line).
usage: python tools/graph_ab.py CONFIG K"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2312_08656_b200 import maxk  # noqa: E402
from paper_2312_08656_b200.layer import MaxkAggregation  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
cfg = synth.CONFIGS[name]
g = synth.config_graph(name)
dev = torch.device("cuda")
agg = MaxkAggregation(*(torch.from_numpy(a).to(dev) for a in (g.row_ptr, g.col_idx, g.val)), cfg.n, cfg.h, k)
x = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.X_SEED)).to(dev)
dy = torch.from_numpy(synth.normal_f32((cfg.n, cfg.h), synth.DY_SEED)).to(dev)
for _ in range(3):
    agg.step(x, dy)
torch.cuda.synchronize()
y_ref, d_ref = agg.y.clone(), agg.d_sp_data.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
graph = torch.cuda.CUDAGraph()
n0 = maxk.launch_count()
with torch.cuda.graph(graph, stream=s):
    agg.step(x, dy)
per = maxk.launch_count() - n0
torch.cuda.synchronize()


def timed(fn, reps=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


te = timed(lambda: agg.step(x, dy))
tg = timed(graph.replay)
ok_y = torch.equal(agg.y, y_ref)  # forward is deterministic
err_d = (agg.d_sp_data - d_ref).abs().max().item()
print(f"{name} k={k}: eager {te:.4f} ms, graph {tg:.4f} ms ({per} kernels per pass); Y bit-identical {ok_y}, "
      f"max |dXs diff| {err_d:.2e}")
