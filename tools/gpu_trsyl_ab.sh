#!/bin/bash
mkdir -p gpurun_out
tag=${1:-ab}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_bs.py -m gpu -q -x > gpurun_out/${tag}_trsyl_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_trsyl_tests.log
for mode in f32 f64; do python tools/trsyl_only.py 4096 $mode 4 >> gpurun_out/${tag}_trsyl_time.log 2>&1; done
python tools/trsyl_only.py 2048 c64 3 >> gpurun_out/${tag}_trsyl_time.log 2>&1
