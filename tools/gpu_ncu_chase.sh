#!/bin/bash
# one full ncu capture (with source counters) of chase_kernel and schur_mss_kernel launches in a 4096 Schur
mkdir -p gpurun_out
tag=${1:-r2}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"${KRE:-chase_kernel}" \
  --launch-skip ${KSKIP:-200} --launch-count ${KCOUNT:-2} -o gpurun_out/${tag}_chase_full -f python tools/schur_only.py 4096 f32 1 > gpurun_out/${tag}_chase_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_chase_ncu.log
