for d in 0 1 2 3; do MSY_TRSYL_DBG=$d timeout 300 python tools/trsyl_only.py 4096 f64 3; done
for d in 0 1 2 3; do MSY_TRSYL_DBG=$d timeout 300 python tools/trsyl_only.py 4096 f32 3; done
