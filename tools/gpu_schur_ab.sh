#!/bin/bash
# Schur correctness tests + 4096 timing (phase breakdown) for an A/B of the Schur kernels
mkdir -p gpurun_out
tag=${1:-ab}
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "schur" > gpurun_out/${tag}_schur_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_schur_tests.log
MSY_SCHUR_TIMING=1 python tools/schur_only.py 4096 f32 3 > gpurun_out/${tag}_schur_time.log 2>&1
python tools/schur_only.py 4096 f32 3 >> gpurun_out/${tag}_schur_time.log 2>&1
python tools/schur_only.py 2048 c64 2 >> gpurun_out/${tag}_schur_time.log 2>&1
