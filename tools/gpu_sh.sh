timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
for c in 4 5; do echo "== CHAINS $c"; MSY_CHAINS=$c timeout 600 python tools/probe.py big 2>&1 | grep "^ch"; done
for t in 1e-2 3e-2; do echo "== SHIFT_TOL $t"; MSY_SHIFT_TOL=$t timeout 600 python tools/probe.py big 2>&1 | grep "^ch"; done
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
