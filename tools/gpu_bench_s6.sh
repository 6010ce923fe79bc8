timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/i_bench_ch.json 2>/dev/null; echo "ch $?"
timeout 900 python bench.py --variant bs --no-cpu-baseline > gpurun_out/i_bench_bs.json 2>/dev/null; echo "bs $?"
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/i_bench_c4.json 2>/dev/null; echo "c4 $?"
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > gpurun_out/i_bench_$c.json; echo "$c $?"; done
