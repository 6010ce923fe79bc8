#!/bin/bash
for dbg in 0 32; do echo "dbg=$dbg" >> gpurun_out/$1.log; MSY_TRSYL_DBG=$dbg python tools/trsyl_only.py 4096 f64 2 >> gpurun_out/$1.log 2>&1; MSY_TRSYL_DBG=$dbg python tools/trsyl_only.py 300 f64 2 >> gpurun_out/$1.log 2>&1; done
