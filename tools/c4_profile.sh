#!/bin/bash
# C4 diagnostics: one m=512 solve alone (phase times), and the launch list of one solve.
mkdir -p gpurun_out
T=${1:-c4p}
python tools/solve_once.py c0 512 512 5 > gpurun_out/${T}_single.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/solve_once.py c0 512 512 1 > /dev/null 2>&1
