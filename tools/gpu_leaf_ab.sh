#!/bin/bash
mkdir -p gpurun_out
tag=${1:-leaf}
for lib in libmpsylv_b200 libmpsylv_leaf1 libmpsylv_leaf2; do
  for mode in f32 f64; do
    echo "$lib" >> gpurun_out/${tag}_time.log
    MSY_LIB_PATH=paper_2503_03456_b200/$lib.so python tools/trsyl_only.py 4096 $mode 4 >> gpurun_out/${tag}_time.log 2>&1
  done
done
