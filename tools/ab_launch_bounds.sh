#!/bin/bash
# A/B of __launch_bounds__ min-blocks for one aggregation kernel (rebuilds libmaxk.so on the box per variant).
# usage: bash tools/ab_launch_bounds.sh KERNEL "0 3 4" "reddit:32 products:32"    (0 = no min-blocks)
kern=${1:-spgemm_fwd_vec_kernel}; variants=${2:-"0 3 4"}; cfgs=${3:-"reddit:32 products:32 flickr:32"}
src=paper_2312_08656_b200/csrc/aggregate_vec.cu
cp $src /tmp/orig_av.cu
for mb in $variants; do
  cp /tmp/orig_av.cu $src
  if [ "$mb" != 0 ]; then
    sed -i -E "s/__launch_bounds__\(VEC_THREADS(, [0-9]+)?\) $kern/__launch_bounds__(VEC_THREADS, $mb) $kern/" $src
  else
    sed -i -E "s/__launch_bounds__\(VEC_THREADS(, [0-9]+)?\) $kern/__launch_bounds__(VEC_THREADS) $kern/" $src
  fi
  python paper_2312_08656_b200/build.py --force > /dev/null
  echo "== $kern minBlocks $mb"
  bash tools/quick_times.sh $cfgs
done
cp /tmp/orig_av.cu $src
python paper_2312_08656_b200/build.py --force > /dev/null
