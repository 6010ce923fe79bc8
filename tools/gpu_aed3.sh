for nw in 64 80 96 112; do MSY_AED_NW=$nw timeout 300 python tools/schur_check.py 4096 f32 2; done
MSY_AED_NW=96 MSY_AED_NIBBLE=25 timeout 300 python tools/schur_check.py 4096 f32 2
MSY_AED_NW=64 MSY_AED_NIBBLE=25 timeout 300 python tools/schur_check.py 4096 f32 2
