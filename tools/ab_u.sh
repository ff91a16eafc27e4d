#!/bin/bash
# A/B of the warp steps in flight of the NC = 16 forward (MAXK_FWD_REP_U): builds the variants, then per-stage times.
# (ptxas keeps ~4-5 steps of gathers in flight whatever U is at k = 32)
for u in 2 8; do python paper_2312_08656_b200/build.py --variant=u$u --define=MAXK_FWD_REP_U=$u > /dev/null; done
for lib in "" paper_2312_08656_b200/libmaxk_u8.so paper_2312_08656_b200/libmaxk_u2.so; do
  echo "== lib=${lib:-default}"
  MAXK_LIB=$lib bash tools/quick_times.sh reddit:32 reddit:64 proteins:32
done
