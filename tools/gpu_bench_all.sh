# round-1 session-2 measurement set: bench lines (CH, BS comparator, C4, reference arm),
# the bench's ncu launch list, and ncu --set full captures of the dominant kernel class
timeout 900 python bench.py > gpurun_out/s2_bench_ch.json 2> gpurun_out/s2_bench_ch.err; echo "ch $?"
timeout 900 python bench.py --variant bs --no-cpu-baseline > gpurun_out/s2_bench_bs.json 2> gpurun_out/s2_bench_bs.err; echo "bs $?"
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s2_bench_c4.json 2> gpurun_out/s2_bench_c4.err; echo "c4 $?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/s2_bench_ref.json 2> gpurun_out/s2_bench_ref.err; echo "ref $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launches_bench_ch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s2_ncu_bench.log 2>&1; echo "ncu list $?"
timeout 900 ncu --set full --clock-control none -k regex:apply_z_multi --launch-skip 400 -c 6 -o /tmp/ncu_az python tools/solve_once.py ch 4096 4096 1 > gpurun_out/s2_ncu_az.log 2>&1; echo "ncu az $?"
ncu -i /tmp/ncu_az.ncu-rep --page raw --csv > gpurun_out/s2_ncu_az_raw.csv 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gemm_dmma --launch-skip 20 -c 2 -o /tmp/ncu_dm python tools/solve_once.py ch 4096 4096 1 > gpurun_out/s2_ncu_dm.log 2>&1; echo "ncu dm $?"
ncu -i /tmp/ncu_dm.ncu-rep --page raw --csv > gpurun_out/s2_ncu_dm_raw.csv 2>&1
