"""Turn the outputs of tools/profile_r02.sh + bench.py + tools/gpu_sweep.sh (gpurun_out/) into the committed round
evidence under profiles/<round>/: launch list + summary, bench line, sweep, ncu --set full summaries with top stall
sites of every captured kernel; merges the per-launch counters into profiles/ncu_counters.json (read by bench.py's
roofline) and the DRAM bytes into profiles/ncu_traffic.json.
usage: python tools/make_round_profiles.py ROUND [BENCH_JSON] [SWEEP_JSONL]"""
import glob
import json
import os
import shutil
import subprocess
import sys

rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", rnd)
bench_src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(G, "bench_default.json")
sweep_src = sys.argv[3] if len(sys.argv) > 3 else os.path.join(G, f"sweep_{rnd}.jsonl")
os.makedirs(P, exist_ok=True)

shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"launches_{rnd}.csv"))
summary = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), os.path.join(G, "launches.csv"),
                          f"{rnd} (bench.py --steps 2 --warmup 3 --e2e-steps 1, Reddit-shaped k=32)"],
                         capture_output=True, text=True).stdout
bench = json.loads(open(bench_src).read().strip().splitlines()[-1])
st = bench["stages_ms"]
summary += (f"\nbench.py (CUDA events, same build, profiles/{rnd}/bench_{rnd}.json): {bench['value']:.2f} ms per step; "
            f"fwd {st['fwd']:.2f}, bwd {st['bwd']:.2f}, top-k {st['topk']:.3f} ms — the shares agree.\n")
open(os.path.join(P, "launches_summary.md"), "w").write(summary)
json.dump(bench, open(os.path.join(P, f"bench_{rnd}.json"), "w"), indent=1)
if os.path.exists(sweep_src):
    shutil.copy(sweep_src, os.path.join(P, f"sweep_{rnd}.jsonl"))

out = [f"# ncu --set full, {rnd} build (one launch per kernel, `--clock-control none`, + lts__t_sectors_op_red/atom)", "",
       "Captured by `tools/profile_r02.sh` (tools/run_stage.py CONFIG K STAGE, the layer path's layouts: the CBSR pair",
       "layout at k = 8 / 16). time_ms is under the profiler (serialised, replayed): shares, not bench numbers.",
       "Per-launch counters of the same captures: profiles/ncu_counters.json (read by bench.py's roofline).", ""]
traffic = {"_source": f"profiles/{rnd}/ncu_{rnd}_summary.md (ncu --set full, dram__bytes_read.sum + "
                      "dram__bytes_write.sum per launch)"}
for path in sorted(glob.glob(os.path.join(G, "sum_*.txt"))):
    tag = os.path.basename(path)[4:-4]
    if not any(tag.startswith(c) for c in ("reddit", "products", "proteins", "flickr")):
        continue  # scratch captures
    lines = open(path).read().splitlines()
    out += [f"## {tag}", ""] + [l for l in lines if l.startswith("|")] + [""]
    for l in lines:
        if l.startswith("{"):
            traffic.update(json.loads(l))
    hot = os.path.join(G, f"hot_{tag}.txt")
    if os.path.exists(hot):
        out += ["Top SASS stall sites (share of warp-stall samples; tools/ncu_hot.py):", "```"]
        out += [l[:110] for l in open(hot).read().splitlines()[1:9]] + ["```", ""]
open(os.path.join(P, f"ncu_{rnd}_summary.md"), "w").write("\n".join(out) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)

cnt_new = os.path.join(G, "ncu_counters.json")
if os.path.exists(cnt_new):
    cnt_path = os.path.join(ROOT, "profiles", "ncu_counters.json")
    cnt = json.load(open(cnt_path)) if os.path.exists(cnt_path) else {}
    cnt.update(json.load(open(cnt_new)))
    json.dump(cnt, open(cnt_path, "w"), indent=1)
print(summary)
