timeout 300 python tools/trsyl_only.py 4096 f64 2 > gpurun_out/trsyl_plain.log 2>&1
for skip in 60 126; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsyl_step --launch-skip $((127+skip)) -c 1 -o /tmp/ncu_trsyl_$skip python tools/trsyl_only.py 4096 f64 2 > gpurun_out/ncu_trsyl_$skip.log 2>&1
ncu -i /tmp/ncu_trsyl_$skip.ncu-rep --page details --csv > gpurun_out/ncu_trsyl_${skip}_details.csv 2>&1
ncu -i /tmp/ncu_trsyl_$skip.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_trsyl_${skip}_source.csv 2>&1
ncu -i /tmp/ncu_trsyl_$skip.ncu-rep --page raw --csv > gpurun_out/ncu_trsyl_${skip}_raw.csv 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:trsyl_step --csv --log-file gpurun_out/trsyl_launches.csv python tools/trsyl_only.py 4096 f64 1 > /dev/null 2>&1
