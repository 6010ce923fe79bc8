for L in libmpsylv_b200.so libmpsylv_hnb24.so libmpsylv_hnb48.so libmpsylv_hnb64.so; do
  echo "== $L"
  MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L MSY_SCHUR_TIMING=1 timeout 300 python tools/schur_check.py 4096 f32 2 2>&1 | grep -v "hess 1[23][0-9]\.[0-9] ms, scan [0-9.]*, small [0-9.]*, shift [0-9.]*, sweep [0-9.]*, aed 0.0 | qr sweeps 1[0-9][0-9], aed windows 0 deflating 0$" | tail -3
  MSY_LIB_PATH=$PWD/paper_2503_03456_b200/$L timeout 600 python tools/probe.py big 2>&1 | grep "^ch"
done
