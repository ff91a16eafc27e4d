#!/bin/bash
# Round-2 evidence on one GPU (outputs in gpurun_out/): ncu --set full (+ L2 reduction sectors) of every step kernel
# on Reddit- and products-shaped graphs at k=32 (+ Reddit k=8 forward), per-launch counters for bench.py's roofline
# (gpurun_out/ncu_counters.json -> profiles/ncu_counters.json), summaries and top stall sites; the ncu launch list
# of the bench command; the bench line itself.
export NCU_COUNTERS_OUT=gpurun_out/ncu_counters.json
X="--metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum"
cap() {  # tag cfg k stage regex
  timeout 900 ncu --set full $X --clock-control none -k "regex:$5" -s 1 -c 1 \
    -o gpurun_out/ncu_$1 python tools/run_stage.py $2 $3 $4 2 > gpurun_out/ncu_$1.log 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_$1.ncu-rep > gpurun_out/sum_$1.txt 2>&1
  python tools/ncu_hot.py gpurun_out/ncu_$1.ncu-rep 25 > gpurun_out/hot_$1.txt 2>&1
  python tools/ncu_counters.py gpurun_out/ncu_$1.ncu-rep $2:k$3:$4 --source "profiles/r02 ncu_$1 (ncu --set full, tools/profile_r02.sh)" >> gpurun_out/counters.log 2>&1
}
for cfg in reddit products; do
  cap ${cfg}_topk $cfg 32 topk topk
  cap ${cfg}_fwd $cfg 32 fwd spgemm_fwd
  cap ${cfg}_bwd $cfg 32 bwd sspmm_bwd
done
cap reddit8_fwd reddit 8 fwd spgemm_fwd
cap reddit16_fwd reddit 16 fwd spgemm_fwd
cap reddit16_topk reddit 16 topk topk
cap reddit8_bwd reddit 8 bwd sspmm_bwd
cap reddit64_fwd reddit 64 fwd spgemm_fwd
for st in topk fwd bwd; do cap flickr_$st flickr 32 $st "topk|spgemm|sspmm"; done
# the fused Eq. 1 kernel (f4) on Reddit-shaped rows (tools/time_f4.py: f = h = 256, k = 32)
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:linear_topk" -s 2 -c 1 \
  -o gpurun_out/ncu_reddit_f4 python tools/time_f4.py > gpurun_out/ncu_reddit_f4.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_reddit_f4.ncu-rep > gpurun_out/sum_reddit_f4.txt 2>&1
python tools/ncu_hot.py gpurun_out/ncu_reddit_f4.ncu-rep 25 > gpurun_out/hot_reddit_f4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
# keep only the Reddit forward report (the others are large)
for f in gpurun_out/ncu_*.ncu-rep; do [ "$f" != "gpurun_out/ncu_reddit_fwd.ncu-rep" ] && rm -f "$f"; done
ls -la gpurun_out | tail -40
