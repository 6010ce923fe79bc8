timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3_pytest.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/r3_pytest.log
timeout 600 python bench.py > gpurun_out/r3_bench_ch.json 2> gpurun_out/r3_bench_ch.err; echo "bench $?"
timeout 600 python bench.py --variant bs --no-cpu-baseline > gpurun_out/r3_bench_bs.json 2> gpurun_out/r3_bench_bs.err; echo "bench bs $?"
MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f64 1 c 2>&1 | tail -3
