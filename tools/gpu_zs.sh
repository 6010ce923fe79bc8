timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -E "^schur|kernels|^m=" | tail -3 | cut -c1-200
MSY_CHASE_ZSPLIT=0 MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -E "^schur|kernels|^m=" | tail -3 | cut -c1-200
timeout 600 python tools/probe.py big 2>&1 | grep -v "^schur"
MSY_CHASE_ZSPLIT=0 timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
