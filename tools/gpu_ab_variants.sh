#!/bin/bash
# A/B of library variants built by tools/build_variant.sh: Schur(4096) alone (time + accuracy) and one CH solve each
mkdir -p gpurun_out
tag=$1; shift
for v in "$@"; do
  lib=$PWD/gpurun_ab/libmpsylv_b200_$v.so
  [ "$v" = base ] && lib=$PWD/paper_2503_03456_b200/libmpsylv_b200.so
  echo "== $v" >> gpurun_out/${tag}_ab.log
  MSY_LIB_PATH=$lib timeout 300 python tools/schur_only.py 4096 f32 3 >> gpurun_out/${tag}_ab.log 2>&1
  MSY_LIB_PATH=$lib timeout 300 python tools/schur_check.py 4096 f32 1 2>&1 | tail -1 | sed "s/env=.*}: //" >> gpurun_out/${tag}_ab.log
  MSY_LIB_PATH=$lib timeout 300 python tools/solve_once.py ch 4096 4096 3 >> gpurun_out/${tag}_ab.log 2>&1
done
