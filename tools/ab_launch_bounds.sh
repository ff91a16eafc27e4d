set -e
cp paper_2312_08656_b200/csrc/aggregate_vec.cu /tmp/orig.cu
for mb in 0 3 4; do
  cp /tmp/orig.cu paper_2312_08656_b200/csrc/aggregate_vec.cu
  if [ $mb != 0 ]; then sed -i "s/__global__ void __launch_bounds__(VEC_THREADS) spgemm_fwd_vec_kernel/__global__ void __launch_bounds__(VEC_THREADS, $mb) spgemm_fwd_vec_kernel/" paper_2312_08656_b200/csrc/aggregate_vec.cu; fi
  python paper_2312_08656_b200/build.py --force > /dev/null
  echo "== minBlocks $mb"
  bash tools/quick_times.sh reddit:32 products:32 flickr:32 reddit:8 reddit:64
done
cp /tmp/orig.cu paper_2312_08656_b200/csrc/aggregate_vec.cu
