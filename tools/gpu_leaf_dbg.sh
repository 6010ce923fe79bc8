#!/bin/bash
mkdir -p gpurun_out
tag=${1:-ld}
for dbg in 0 4 8 12 16 28; do
  echo "dbg=$dbg" >> gpurun_out/${tag}.log
  MSY_TRSYL_DBG=$dbg python tools/trsyl_only.py 4096 f64 3 >> gpurun_out/${tag}.log 2>&1
done
