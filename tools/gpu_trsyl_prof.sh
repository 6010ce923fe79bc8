#!/bin/bash
mkdir -p gpurun_out
tag=${1:-tl}
for mode in f32 f64; do python tools/trsyl_only.py 4096 $mode 4 >> gpurun_out/${tag}_trsyl_time.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_trsyl_launches.csv python tools/trsyl_only.py 4096 f64 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_bs.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/${tag}_trsyl_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_trsyl_tests.log
