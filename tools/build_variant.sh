#!/bin/bash
# A/B build: tools/build_variant.sh NAME -DMSY_X=... -> gpurun_ab/libmpsylv_b200_NAME.so (select with MSY_LIB_PATH)
name=$1; shift
mkdir -p gpurun_ab
cd paper_2503_03456_b200
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -diag-suppress 177 "$@" -o ../gpurun_ab/libmpsylv_b200_$name.so csrc/solver.cu
