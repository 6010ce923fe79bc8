#!/bin/bash
mkdir -p gpurun_out
tag=${1:-aed}
for nw in 128 96 64; do
  echo "AED nw=$nw" >> gpurun_out/${tag}.log
  MSY_AED=1 MSY_AED_NW=$nw MSY_SCHUR_TIMING=1 python tools/schur_only.py 4096 f32 2 >> gpurun_out/${tag}.log 2>&1
done
echo "no AED" >> gpurun_out/${tag}.log
MSY_SCHUR_TIMING=1 python tools/schur_only.py 4096 f32 2 >> gpurun_out/${tag}.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv env MSY_AED=1 python tools/schur_only.py 4096 f32 1 > /dev/null 2>&1
