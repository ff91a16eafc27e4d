#!/bin/bash
# Round evidence on one GPU: bench line, ncu launch list of the bench command, one ncu --set full capture of
# each step kernel (Reddit- and products-shaped, k=32), and the per-config sweep.  Outputs in gpurun_out/.
set -x
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log > gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
for cfg in reddit products; do
  for st in topk fwd bwd; do
    case $st in topk) kr="regex:topk";; fwd) kr="regex:spgemm_fwd_vec";; bwd) kr="regex:sspmm_bwd_vec";; esac
    timeout 600 ncu --set full --import-source on --clock-control none -k "$kr" -s 1 -c 1 \
      -o gpurun_out/full_${cfg}_${st} python tools/run_stage.py $cfg 32 $st 1 > /dev/null 2>&1
  done
done
bash tools/gpu_sweep.sh gpurun_out/sweep.jsonl 20
# summaries on the box (the .ncu-rep files are large): keep the Reddit forward report only
for cfg in reddit products; do
  for st in topk fwd bwd; do
    python tools/ncu_summary.py gpurun_out/full_${cfg}_${st}.ncu-rep --traffic-key ${cfg}:k32 > gpurun_out/sum_${cfg}_${st}.txt 2>&1
    python tools/ncu_hot.py gpurun_out/full_${cfg}_${st}.ncu-rep 25 > gpurun_out/hot_${cfg}_${st}.txt 2>&1
    ncu -i gpurun_out/full_${cfg}_${st}.ncu-rep --page raw --csv > gpurun_out/raw_${cfg}_${st}.csv 2>/dev/null
    [ "$cfg/$st" != "reddit/fwd" ] && rm -f gpurun_out/full_${cfg}_${st}.ncu-rep
  done
done
ls -la gpurun_out
