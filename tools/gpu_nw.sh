for L in libmpsylv_b200.so libmpsylv_nw12.so libmpsylv_nw16.so; do
  echo "== $L"
  MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -E "^schur|^m=" | tail -2 | cut -c1-180
  for m in 100 128; do MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L timeout 120 python tools/schur_check.py $m f32 2 2>&1 | grep "^m=" | cut -c1-40,150-260; done
  MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L timeout 600 python tools/probe.py big 2>&1 | grep "^ch" | cut -c1-60,140-260
done
