#!/bin/bash
# Round measurement package: GPU tests, bench lines for every config, the CH launch list and
# one ncu --set full capture per dominant kernel.  Everything lands in gpurun_out/TAG_*.
mkdir -p gpurun_out
T=${1:-r2m}
timeout 2400 python -m pytest tests -m gpu -q -rs -p no:cacheprovider > gpurun_out/${T}_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_gputest.log
python bench.py > gpurun_out/${T}_bench_ch.log 2>&1
python bench.py --correction 32 --no-c4 > gpurun_out/${T}_bench_ch32.log 2>&1
python bench.py --variant bs --no-c4 --no-cpu-baseline > gpurun_out/${T}_bench_bs.log 2>&1
for c in c0 c1 c2 c3; do python bench.py --config $c --steps 5 > gpurun_out/${T}_bench_$c.log 2>&1; done
python bench.py --config c4 > gpurun_out/${T}_bench_c4.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_ch.csv python tools/solve_once.py ch 4096 4096 > /dev/null 2>&1
for spec in "chase_kernel:900" "apply_z_cl_kernel:3000" "hess_panel2_kernel:60" "schur_mss_kernel:40" "trsyl_step_kernel:60" "trsyl_lpart_dmma_kernel:200" "gemm_dmma_kernel:30" "rankk_update_kernel:100" "vtc_partial_kernel:100"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip $s --launch-count 1 -o gpurun_out/${T}_full_$k -f python tools/solve_once.py ch 4096 4096 > gpurun_out/${T}_full_$k.log 2>&1
done
