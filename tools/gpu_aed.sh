# AED experiments: Schur accuracy/timing at several sizes and settings, then the GPU tests
export MSY_SCHUR_TIMING=1
for m in 200 512 1024; do timeout 120 python tools/schur_check.py $m f32 2; done
timeout 120 python tools/schur_check.py 512 c64 2
timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED=0 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED_GMAX=4 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED_GMAX=48 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED_GMAX=128 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED_NIBBLE=30 timeout 300 python tools/schur_check.py 4096 f32 2
timeout 300 python tools/schur_check.py 2048 c64 2
MSY_AED=0 timeout 300 python tools/schur_check.py 2048 c64 2
unset MSY_SCHUR_TIMING
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python tools/probe.py big
