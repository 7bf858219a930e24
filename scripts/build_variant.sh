#!/bin/bash
# A/B variant of the library with extra nvcc defines -> scripts/_timing/<name>.so
# usage: scripts/build_variant.sh <name> -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/var_$name scripts/_timing
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -diag-suppress 39,177,550,186 $*"
objs=""
for s in kernels_1d kernels_mv kernels_large kernels_2d kernels_full kernels_krylov kernels_commuted kernels_tsplit api; do
  nvcc $F -c paper_2003_07020_b200/csrc/$s.cu -o build/var_$name/$s.o &
  objs="$objs build/var_$name/$s.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/_timing/$name.so $objs
