#!/bin/bash
# Schur(4096) phase breakdown and per-kernel launch list (ncu, serialised, cold-cache).
mkdir -p gpurun_out
tag=${1:-r2}
MSY_SCHUR_TIMING=1 python tools/schur_only.py 4096 f32 3 > gpurun_out/${tag}_schur_phases.log 2>&1
python tools/schur_only.py 4096 f32 3 >> gpurun_out/${tag}_schur_phases.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_schur_launches.csv \
  python tools/schur_only.py 4096 f32 1 > gpurun_out/${tag}_schur_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_schur_ncu.log
