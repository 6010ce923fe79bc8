set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s2_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/r1s2_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r1s2_bench_ch.json 2> gpurun_out/r1s2_bench_ch.err; echo "bench exit $?"
cat gpurun_out/r1s2_bench_ch.json
timeout 600 python tools/probe.py big > gpurun_out/r1s2_probe_big.log 2>&1; echo "probe exit $?"
cat gpurun_out/r1s2_probe_big.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s2_launches_ch.csv python tools/solve_once.py ch 4096 4096 2 > gpurun_out/r1s2_ncu_launch.log 2>&1; echo "ncu exit $?"
