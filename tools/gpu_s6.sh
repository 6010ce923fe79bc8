timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/g_bench_ch.json 2>/dev/null; echo "ch $?"
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench_c4.json 2>/dev/null; echo "c4 $?"
timeout 900 python bench.py --variant bs --no-cpu-baseline > gpurun_out/g_bench_bs.json 2>/dev/null; echo "bs $?"
for c in c1 c2 c3; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', round(d['value'],3), round(d['ms_per_step'],1), d['config']['iterations'], d['config']['backward_error'])"; done
