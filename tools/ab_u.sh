for lib in "" paper_2312_08656_b200/libmaxk_u8.so paper_2312_08656_b200/libmaxk_u6.so paper_2312_08656_b200/libmaxk_u2.so; do
  echo "== lib=${lib:-default}"
  MAXK_LIB=$lib bash tools/quick_times.sh reddit:32 reddit:64 proteins:32
done
