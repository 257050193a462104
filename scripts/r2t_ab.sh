#!/bin/bash
O=gpurun_out/${1:-r2t}
mkdir -p $O
export NLFEM_GPU_LIB=$PWD/paper_2302_07499_b200/libnlfem_gpu_nored.so
MODES="1 0" CONFIGS="C4" bash scripts/r2s_ab.sh $1
