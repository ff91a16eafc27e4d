#!/bin/bash
# The bench line's `parity` block (outputs of the timed run vs the fp64 oracle) on every BASELINE.json config, with a
# CPU budget large enough for all rows where the oracle finishes (one JSON line per config/k).
out=${1:-gpurun_out/parity_all_configs.jsonl}
: > "$out"
for ck in tiny:8 flickr:16 flickr:32 flickr:64 proteins:32 reddit:8 reddit:16 reddit:32 reddit:64 products:32; do
  c=${ck%%:*}; k=${ck##*:}
  timeout 900 python bench.py --config "$c" --k "$k" --steps 5 --warmup 3 --e2e-steps 1 --cpu-budget-s 60 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config': '$c', 'k': $k, 'ms': d['value'], 'parity': d.get('parity'), 'cpu_baseline': {kk: d['cpu_baseline'].get(kk) for kk in ('value', 'cores', 'sample')}}))" >> "$out" \
    || echo "{\"config\": \"$c\", \"k\": $k, \"failed\": true}" >> "$out"
done
