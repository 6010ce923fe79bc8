export MSY_SCHUR_TIMING=1
timeout 300 python tools/schur_check.py 4096 f32 2
for nb in 16 12 8; do MSY_NB=$nb timeout 300 python tools/schur_check.py 4096 f32 2; done
MSY_NB=12 MSY_CHAINS=6 timeout 300 python tools/schur_check.py 4096 f32 2
unset MSY_SCHUR_TIMING
for nb in 24 16 12; do MSY_NB=$nb timeout 300 python tools/probe.py big 2>&1 | grep "^ch"; done
