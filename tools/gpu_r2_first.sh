#!/bin/bash
# round-2 first GPU call: box CPU inventory, GPU tests, default bench line
mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g) > gpurun_out/r2_box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_gputest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_ch.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench_ch.log
