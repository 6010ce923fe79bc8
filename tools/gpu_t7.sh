for t in f32 f64; do timeout 300 python tools/trsyl_only.py 4096 $t 3; done
for t in c64 c128; do timeout 300 python tools/trsyl_only.py 2048 $t 3; done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python tools/probe.py big 2>&1 | grep -v "^schur"
