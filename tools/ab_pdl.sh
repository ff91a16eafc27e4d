#!/bin/bash
# A/B of programmatic dependent launch (MAXK_PDL=0 vs default) on the layer pass: device-timed ms per step.
for pdl in 0 1; do
  echo "== MAXK_PDL=$pdl"
  MAXK_PDL=$pdl bash tools/quick_times.sh tiny:8 flickr:16 flickr:32 flickr:64 reddit:32 products:32
done
