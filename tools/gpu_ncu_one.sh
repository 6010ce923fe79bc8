#!/bin/bash
# one full ncu capture (source counters) of launches matching KRE, skipping KSKIP, of CMD
mkdir -p gpurun_out
tag=${1:-r2}
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"${KRE}" \
  --launch-skip ${KSKIP:-0} --launch-count ${KCOUNT:-1} -o gpurun_out/${tag} -f ${CMD} > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu.log
