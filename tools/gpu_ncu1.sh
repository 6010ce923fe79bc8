for k in schur_mss_kernel aed_kernel chase_kernel apply_z_multi_kernel; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 20 -c 1 -o /tmp/ncu_$k python tools/schur_check.py 4096 f32 1 > gpurun_out/ncu_$k.log 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page details --csv > gpurun_out/ncu_${k}_details.csv 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page source --csv > gpurun_out/ncu_${k}_source.csv 2>&1
ncu -i /tmp/ncu_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>&1
done
ls -la gpurun_out
