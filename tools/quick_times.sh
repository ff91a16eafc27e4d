#!/bin/bash
# Per-kernel device times for a few configs (quick A/B check; not the driver's bench line).
# usage: bash tools/quick_times.sh [configs...]   e.g. reddit:32 products:32 flickr:32
cfgs=${*:-reddit:32 products:32 flickr:32}
for ck in $cfgs; do
  c=${ck%%:*}; k=${ck##*:}
  timeout 600 python bench.py --config "$c" --k "$k" --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
    2>/dev/null | tail -1 > gpurun_out/qt.out
  python - "$ck" <<'PY'
import json, sys
d = json.load(open("gpurun_out/qt.out"))
kt = d.get("stages_ms", {})
print(sys.argv[1], "ms %.3f" % d["ms_per_step"], " ".join("%s %.3f" % (n, v) for n, v in kt.items()))
PY
done
