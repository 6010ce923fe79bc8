#!/bin/bash
# default bench line (+ optional extra args), log under gpurun_out/
mkdir -p gpurun_out
tag=${1:-b}
shift
timeout 1500 python bench.py "$@" > gpurun_out/${tag}_bench.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_bench.log
