#!/bin/bash
# Round measurement package, part 1: GPU tests, bench lines for every config, the CH launch
# list, the full-size parity table.  Everything lands in gpurun_out/TAG_* (small files).
mkdir -p gpurun_out
T=${1:-r2m}
timeout 2400 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/${T}_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gputest.log
python tools/parity_table.py gpurun_out/${T}_parity.json > gpurun_out/${T}_parity.log 2>&1
python bench.py > gpurun_out/${T}_bench_ch.log 2>&1
python bench.py --correction 32 --no-c4 > gpurun_out/${T}_bench_ch32.log 2>&1
python bench.py --variant bs --no-c4 --no-cpu-baseline > gpurun_out/${T}_bench_bs.log 2>&1
for c in c0 c1 c2 c3; do python bench.py --config $c --steps 5 > gpurun_out/${T}_bench_$c.log 2>&1; done
python bench.py --config c4 > gpurun_out/${T}_bench_c4.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.log 2>&1
python bench.py --impl reference --config c0 --steps 1 --warmup 0 > gpurun_out/${T}_bench_ref_c0.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_ch.csv python tools/solve_once.py ch 4096 4096 > /dev/null 2>&1
