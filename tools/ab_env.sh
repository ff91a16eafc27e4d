#!/bin/bash
# A/B per-stage device times over env settings: bash tools/ab_env.sh "VAR=a VAR=b" "reddit:32 products:32"
settings=${1}; cfgs=${2:-"reddit:32 products:32"}
for st in $settings; do
  for ck in $cfgs; do
    c=${ck%%:*}; k=${ck##*:}
    env $st timeout 600 python bench.py --config "$c" --k "$k" --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
      2>/dev/null | tail -1 > gpurun_out/ab.out
    python - "$st" "$ck" <<'PY'
import json, sys
try:
    d = json.load(open("gpurun_out/ab.out"))
except Exception:
    print(sys.argv[1], sys.argv[2], "FAILED"); sys.exit(0)
print(sys.argv[1], sys.argv[2], "ms %.3f" % d["value"], " ".join("%s %.3f" % (k, v) for k, v in d["stages_ms"].items()
                                                          if k in ("topk", "fwd", "bwd")))
PY
  done
done
