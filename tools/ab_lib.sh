#!/bin/bash
# A/B of two builds of the same sources (default libmaxk.so vs $1) on fwd and bwd: tools/ab_lib.sh LIB CASES...
lib=$1; shift
for st in fwd bwd; do
  python tools/ab_fwd.py "$@" --stage $st --modes "MAXK_NONE=0" | sed "s/^/default $st /"
  MAXK_LIB=$lib python tools/ab_fwd.py "$@" --stage $st --modes "MAXK_NONE=0" | sed "s/^/$(basename $lib) $st /"
done
