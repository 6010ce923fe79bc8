for v in base sub1024; do
  lib=$PWD/gpurun_ab/libmpsylv_b200_$v.so
  [ "$v" = base ] && lib=$PWD/paper_2503_03456_b200/libmpsylv_b200.so
  for r in 1 2 3; do MSY_LIB_PATH=$lib python tools/schur_check.py 4096 f32 1 2>&1 | tail -1 | sed 's/env=.*}: //' >> gpurun_out/s4h_chk.log; done
  MSY_LIB_PATH=$lib python tools/schur_check.py 2500 f32 1 2>&1 | tail -1 | sed 's/env=.*}: //' >> gpurun_out/s4h_chk.log
  MSY_LIB_PATH=$lib python tools/schur_check.py 2048 c64 1 2>&1 | tail -1 | sed 's/env=.*}: //' >> gpurun_out/s4h_chk.log
done
