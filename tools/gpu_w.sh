for L in libmpsylv_w128_nb16.so libmpsylv_w128_nb12.so libmpsylv_w112_nb12.so libmpsylv_w144_nb20.so libmpsylv_w96_nb8.so; do
  echo "== $L"
  MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -v "hess 1[23]\|kernels"
  MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
done
