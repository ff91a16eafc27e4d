#!/bin/bash
# ncu --set full capture of one hot-path stage on one config, summarised on the box.
# usage: tools/ncu_stage.sh TAG CONFIG K STAGE KERNEL_REGEX   (env knobs pass through)
tag=$1; cfg=$2; k=$3; st=$4; kr=$5
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:$kr" -s 1 -c 1 \
  -o gpurun_out/ncu_$tag python tools/run_stage.py $cfg $k $st 2 > gpurun_out/ncu_$tag.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$tag.ncu-rep > gpurun_out/sum_$tag.txt 2>&1
python tools/ncu_hot.py gpurun_out/ncu_$tag.ncu-rep 40 > gpurun_out/hot_$tag.txt 2>&1
ncu -i gpurun_out/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv 2>/dev/null
