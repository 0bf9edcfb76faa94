#!/bin/bash
# Build a variant of liblrnr_gpu.so with extra nvcc flags for the meta tensor-core
# TU only (dev aid for timing experiments):  scripts/build_meta_variant.sh NAME -DMTC_SKIP=1
# -> scripts/liblrnr_gpu_NAME.so (load with LRNR_GPU_LIB=...).  Needs the regular build first.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
    --expt-relaxed-constexpr "$@" -c paper_2410_04001_b200/csrc/meta_tc.cu -o build/meta_tc_$name.o
others=$(ls build/*.cu.o | grep -v '/meta_tc.cu.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/liblrnr_gpu_$name.so build/meta_tc_$name.o \
    $others build/*.cpp.o -cudart static
