export MSY_SCHUR_TIMING=1
for g in 0 4 16; do MSY_AED_GMAX=$g timeout 300 python tools/schur_check.py 4096 f32 2; done
MSY_AED=0 timeout 300 python tools/schur_check.py 4096 f32 2
