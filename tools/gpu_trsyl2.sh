for t in c128 c64; do timeout 300 python tools/trsyl_only.py 1024 $t 2; done
timeout 300 python -m pytest tests/test_bs.py -m gpu -x -q 2>&1 | grep -E "Error|error|assert" | head -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:trsyl_step --csv --log-file gpurun_out/trsyl_launches2.csv python tools/trsyl_only.py 4096 f64 1 > /dev/null 2>&1
