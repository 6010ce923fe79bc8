#!/bin/bash
# GPU test pass: the whole -m gpu suite (log under gpurun_out/)
mkdir -p gpurun_out
tag=${1:-r2}
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 -p no:cacheprovider > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
