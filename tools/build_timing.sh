#!/bin/bash
# Timing build of the library (clock64 phase counters in the Jacobi solvers)
# -> tools/libpod_timing.so, used by tools/cj_timing.py and tools/bj_timing.py
set -e
cd "$(dirname "$0")/../paper_1905_05107_b200/csrc"
T=$(mktemp -d)
for f in capi sampling gemm_f64 small cluster_jacobi block_jacobi grid_jacobi misc residual; do
  nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
    -DPOD_CJ_TIMING -DPOD_BJ_TIMING -c $f.cu -o $T/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/libpod_timing.so $T/*.o -lcudart
rm -rf $T
