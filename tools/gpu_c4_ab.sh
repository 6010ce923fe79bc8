#!/bin/bash
# C4 A/B over library variants (tools/build_variant.sh NAME ...): bash tools/gpu_c4_ab.sh TAG NAME...
mkdir -p gpurun_out
tag=${1:-c4ab}; shift
for v in "$@"; do
  lib=$PWD/gpurun_ab/libmpsylv_b200_$v.so
  [ "$v" = base ] && lib=$PWD/paper_2503_03456_b200/libmpsylv_b200.so
  echo "== $v" >> gpurun_out/${tag}.log
  MSY_LIB_PATH=$lib python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['lane_phase_ms_mean'])" >> gpurun_out/${tag}.log 2>&1
done
# lane-count sweep for the last variant: LANES="48 96 128" bash tools/gpu_c4_ab.sh TAG NAME
for ln in $LANES; do
  echo "== $v lanes $ln" >> gpurun_out/${tag}.log
  MSY_LIB_PATH=$lib python bench.py --config c4 --lanes $ln --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['config']['lane_phase_ms_mean'])" >> gpurun_out/${tag}.log 2>&1
done
