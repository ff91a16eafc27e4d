#!/bin/bash
# Backward target-column blocking sweep (bench.py --bwd-blocks) on one config; device-timed per-stage lines.
# usage: bash tools/bwd_blocks_sweep.sh CONFIG "1 0 2 4"
c=${1:-products}; bl=${2:-"1 0 2 3 4 6 8"}
for b in $bl; do
  timeout 300 python bench.py --config "$c" --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --bwd-blocks "$b" \
    2>gpurun_out/sweep_err.log | tail -1 > gpurun_out/sw.out
  python - "$b" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/sw.out"))
except Exception:
    print("blocks", sys.argv[1], "FAILED"); sys.exit(0)
print("blocks arg", sys.argv[1], "used", d["config"]["bwd_blocks"], "ms %.3f" % d["value"],
      " ".join("%s %.3f" % (k, v) for k, v in d["stages_ms"].items()))
PY
done
