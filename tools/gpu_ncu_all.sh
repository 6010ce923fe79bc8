#!/bin/bash
# Round measurement package, part 2: one ncu --set full capture per dominant kernel of a CH
# solve, exported on the box to compact CSV (raw metrics + per-source-line hot spots); the
# .ncu-rep files are deleted (gpurun copies back at most 64 MiB).
mkdir -p gpurun_out
T=${1:-r2n}
mkdir -p /tmp/cub && (cd /tmp/cub && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_2503_03456_b200/libmpsylv_b200.so > /dev/null 2>&1)
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for spec in "chase2_kernel:900" "apply_z_far_kernel:1500" "apply_z_cl_kernel:3000" "hess_panel2_kernel:60" "schur_mss_kernel:40" "trsyl_step_kernel:60" "trsyl_lpart_dmma_kernel:200" "gemm_dmma_kernel:30" "rankk_update_kernel:100" "vtc_partial_kernel:100"; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip $s --launch-count 1 -o /tmp/${T}_$k -f python tools/solve_once.py ch 4096 4096 > /dev/null 2>&1
  ncu -i /tmp/${T}_$k.ncu-rep --page raw --csv --metrics $M > gpurun_out/${T}_$k.raw.csv 2>&1
  python tools/sass_lines.py /tmp/${T}_$k.ncu-rep "$k" /tmp/cub/solver.sm_100a.cubin 25 > gpurun_out/${T}_$k.lines.txt 2>&1
done
ls -la /tmp/*.ncu-rep > gpurun_out/${T}_reps.txt
