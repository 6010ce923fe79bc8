timeout 900 python bench.py > gpurun_out/h_bench_ch.json 2>/dev/null; echo "ch $?"
timeout 900 python bench.py --variant bs --no-cpu-baseline > gpurun_out/h_bench_bs.json 2>/dev/null; echo "bs $?"
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/h_bench_c4.json 2>/dev/null; echo "c4 $?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/h_bench_ref.json 2>/dev/null; echo "ref $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/h_launches_solve.csv python tools/solve_once.py ch 4096 4096 1 > /dev/null 2>&1; echo "ncu list $?"
timeout 900 ncu --set full --clock-control none -k regex:apply_z_cl --launch-skip 400 -c 6 -o /tmp/ncu_azc2 python tools/solve_once.py ch 4096 4096 1 > /dev/null 2>&1; echo "ncu azc $?"
ncu -i /tmp/ncu_azc2.ncu-rep --page raw --csv > gpurun_out/h_ncu_azc_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:chase_kernel --launch-skip 200 -c 2 -o /tmp/ncu_ch2 python tools/solve_once.py ch 4096 4096 1 > /dev/null 2>&1; echo "ncu chase $?"
ncu -i /tmp/ncu_ch2.ncu-rep --page raw --csv > gpurun_out/h_ncu_ch_raw.csv 2>&1
