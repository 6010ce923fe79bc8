export MSY_SCHUR_TIMING=1
for m in 64 100 128; do for w in 0 24; do MSY_MSS_AED=$w timeout 120 python tools/schur_check.py $m f32 2; done; done
for w in 0 16 24 32; do MSY_MSS_AED=$w timeout 120 python tools/schur_check.py 96 c64 2; done
for w in 0 24; do MSY_MSS_AED=$w timeout 120 python tools/schur_check.py 512 f32 2; done
for w in 16 24 32; do MSY_AED=1 MSY_MSS_AED=$w timeout 300 python tools/schur_check.py 4096 f32 2; done
MSY_AED=1 MSY_MSS_AED=24 MSY_MSS_AEDG=2 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED=1 MSY_MSS_AED=24 MSY_MSS_AEDG=16 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED=0 MSY_MSS_AED=24 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED=1 MSY_MSS_AED=24 timeout 300 python tools/schur_check.py 2048 c64 2
unset MSY_SCHUR_TIMING
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
