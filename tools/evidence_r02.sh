#!/bin/bash
# Round-2 evidence refresh on one GPU: ncu captures + per-launch counters + launch list (tools/profile_r02.sh),
# the default bench line, the sweep of every config, then tools/make_round_profiles.py r02 (run here afterwards).
rm -f gpurun_out/sum_*.txt gpurun_out/hot_*.txt gpurun_out/ncu_counters.json gpurun_out/counters.log
bash tools/profile_r02.sh > gpurun_out/profile_r02.log 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
bash tools/gpu_sweep.sh gpurun_out/sweep_r02.jsonl 20
tail -c 600 gpurun_out/bench_default.json
