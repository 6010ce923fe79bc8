#!/bin/bash
# C4 A/B over library builds: MSY_LIB_PATH=... python bench.py --config c4
mkdir -p gpurun_out
tag=${1:-c4ab}; shift
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/${tag}.log
  MSY_LIB_PATH=paper_2503_03456_b200/$lib.so python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['lane_phase_ms_mean'])" >> gpurun_out/${tag}.log 2>&1
done
