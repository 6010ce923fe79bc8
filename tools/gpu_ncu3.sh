timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsyl_step --launch-skip 253 -c 1 -o /tmp/ncu_t python tools/trsyl_only.py 4096 f64 2 > gpurun_out/ncu_t.log 2>&1
ncu -i /tmp/ncu_t.ncu-rep --page details --csv > gpurun_out/ncu_t_details.csv 2>&1
ncu -i /tmp/ncu_t.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_t_source.csv 2>&1
for i in 1 2 3 4 5 6 7 8; do timeout 120 python -m pytest tests/test_bs.py -m gpu -x -q 2>&1 | tail -1; done
