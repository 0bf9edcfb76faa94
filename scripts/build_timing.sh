#!/bin/bash
# Build the library with the tensor-core kernel's per-phase cycle counters
# (-DLRNR_TC_TIMING) into scripts/liblrnr_gpu_timing.so; read with
#   LRNR_GPU_LIB=scripts/liblrnr_gpu_timing.so python scripts/tc_timing.py [fast_sincos]
# Needs the regular build (python -c "import __graft_entry__ as g; g.build()") first.
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
    --expt-relaxed-constexpr -diag-suppress 177 -DLRNR_TC_TIMING "$@" \
    -c paper_2410_04001_b200/csrc/lrnr_gpu.cu -o build/lrnr_gpu_timing.o
others=$(ls build/*.cu.o | grep -v '/lrnr_gpu.cu.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/liblrnr_gpu_timing.so build/lrnr_gpu_timing.o \
    $others build/*.cpp.o -cudart static -ldl
