timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py --variant bs --no-cpu-baseline > gpurun_out/l_bench_bs.json 2>/dev/null; echo "bs $?"
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/l_bench_$c.json; echo "$c $?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/l_launches_solve.csv python tools/solve_once.py ch 4096 4096 1 > /dev/null 2>&1; echo "ncu list $?"
