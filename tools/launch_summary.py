"""Per-kernel table from an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, median ms, and
each step kernel's share of the step (sum of the step kernels' medians).
usage: python tools/launch_summary.py LAUNCHES.csv [TITLE]"""
import csv
import statistics
import sys

STEP = ("topk_cbsr_kernel", "topk_newton_kernel", "topk_fast_kernel", "spgemm_fwd_kernel", "spgemm_fwd_vec_kernel", "sspmm_bwd_vec_kernel", "combine_kernel",
        "zero4_kernel")
lines = open(sys.argv[1]).read().splitlines()
lines = lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]  # skip ncu's ==PROF== preamble
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
by = {}
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("maxk::<unnamed>::", "")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}[r["Metric Unit"]]
    by.setdefault(name, []).append(float(r["Metric Value"].replace(",", "")) * scale)
step = {k: statistics.median(v) for k, v in by.items() if k.split("<")[0] in STEP}
tot = sum(step.values())
print(f"# ncu launch list{': ' + sys.argv[2] if len(sys.argv) > 2 else ''}\n")
print("Per-launch device time from `ncu --metrics gpu__time_duration.sum --clock-control none` (serialised, cold).\n")
print("| kernel | launches | median ms | share of the step |\n|---|---|---|---|")
for k, v in sorted(step.items(), key=lambda x: -x[1]):
    print(f"| {k} | {len(by[k])} | {v:.4f} | {v / tot * 100:.1f}% |")
print(f"| **step (sum of medians)** | | **{tot:.3f}** | 100% |\n")
print("Not part of the step:\n")
for k, v in sorted(by.items(), key=lambda x: -statistics.median(x[1])):
    if k not in step and (k.startswith("cbsr") or k.startswith("linear") or "maxk" in k or "nvjet" in k):
        print(f"- {k}: {len(v)} launches, median {statistics.median(v):.4f} ms")
