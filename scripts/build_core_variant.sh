#!/bin/bash
# Build a variant of liblrnr_gpu.so with extra nvcc flags for lrnr_gpu.cu (the tensor-core
# tile kernel's TU) only (dev aid):  scripts/build_core_variant.sh NAME -DTC_SPLIT_ISSUE=0
# -> scripts/liblrnr_gpu_NAME.so (load with LRNR_GPU_LIB=...).  Needs the regular build first.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
    --expt-relaxed-constexpr "$@" -c paper_2410_04001_b200/csrc/lrnr_gpu.cu -o build/lrnr_gpu_$name.o
others=$(ls build/*.cu.o | grep -v '/lrnr_gpu.cu.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/liblrnr_gpu_$name.so build/lrnr_gpu_$name.o \
    $others build/*.cpp.o -cudart static -ldl
