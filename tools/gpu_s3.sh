timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for a in 0 1 2; do MSY_AZC=$a MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -v "^schur m"; done
for a in 0 1 2; do MSY_AZC=$a timeout 600 python tools/probe.py big 2>&1 | grep "^ch"; done
