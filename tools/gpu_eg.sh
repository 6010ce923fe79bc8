timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -v "hess 1[23]"
MSY_SYNC_ENDGAME=1 MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -v "hess 1[23]"
timeout 300 python tools/schur_check.py 1000 f32 2
timeout 300 python tools/schur_check.py 1000 c64 2
timeout 600 python tools/probe.py big 2>&1 | grep -v "^schur"
MSY_SYNC_ENDGAME=1 timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
