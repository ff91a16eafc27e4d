#!/bin/bash
# compute-sanitizer on the r02 build (outputs in gpurun_out/san_r02c/)
mkdir -p gpurun_out/san_r02c
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_r02c/${tool}.log 2>&1
  echo "$tool: exit $? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' gpurun_out/san_r02c/${tool}.log | tr '\n' ' ')"
done
for tool in memcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py --flickr > gpurun_out/san_r02c/${tool}_flickr.log 2>&1
  echo "$tool flickr: exit $? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run flickr ok' gpurun_out/san_r02c/${tool}_flickr.log | tr '\n' ' ')"
done
