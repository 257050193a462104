#!/bin/bash
# Build paper_2302_07499_b200/libnlfem_gpu_<tag>.so with extra nvcc defines on
# nlfem_gpu.cu (the other objects from the in-tree build): A/B variants timed
# side by side through NLFEM_GPU_LIB.   scripts/build_variant.sh TAG -DX=1 ...
set -e
T=$1; shift
D=paper_2302_07499_b200
B=$D/_build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I include -I $D/csrc "$@" \
  -c $D/csrc/nlfem_gpu.cu -o $B/nlfem_gpu_$T.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $D/libnlfem_gpu_$T.so $B/nlfem_gpu_$T.o \
  $(ls $B/*.o | grep -v -e "/nlfem_gpu.cu.o" -e "/nlfem_gpu_") -lcudart_static -lrt -ldl -lpthread
