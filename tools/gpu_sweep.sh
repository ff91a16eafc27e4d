#!/bin/bash
# Run bench.py over every BASELINE.json config/k on one GPU (device-timed lines; not the driver's bench line).
# usage: bash tools/gpu_sweep.sh OUTFILE [steps]
out=${1:-gpurun_out/sweep.jsonl}; steps=${2:-20}
: > "$out"
for ck in tiny:8 flickr:16 flickr:32 flickr:64 proteins:32 reddit:8 reddit:16 reddit:32 reddit:64 products:32; do
  c=${ck%%:*}; k=${ck##*:}
  timeout 600 python bench.py --config "$c" --k "$k" --steps "$steps" --warmup 3 --e2e-steps 2 --no-cpu-baseline \
    2>/dev/null | tail -1 >> "$out" || echo "{\"config\": \"$c\", \"k\": $k, \"failed\": true}" >> "$out"
done
