#!/bin/bash
# development build with clock64 phase stamps (-DFPC_PHASE_TIMING) -> scripts/_timing/libfpc_timing.so (travels with gpurun; git-ignored)
set -e
cd "$(dirname "$0")/.."
mkdir -p build/timing scripts/_timing
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -diag-suppress 39 -DFPC_PHASE_TIMING"
objs=""
for s in kernels_1d kernels_mv kernels_large kernels_2d kernels_full kernels_krylov kernels_commuted api; do
  nvcc $F -c paper_2003_07020_b200/csrc/$s.cu -o build/timing/$s.o &
  objs="$objs build/timing/$s.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/_timing/libfpc_timing.so $objs
