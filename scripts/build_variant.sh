#!/bin/bash
# A/B variant of the library: recompiles only the named sources with extra nvcc defines and links
# them with the main build's other objects (build/fpc) -> scripts/_timing/<name>.so
# usage: scripts/build_variant.sh <name> "<src1 src2 ...>" -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; srcs=$2; shift 2
mkdir -p build/var_$name scripts/_timing
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-march=x86-64-v3,-ffp-contract=fast --expt-relaxed-constexpr -diag-suppress 39 $*"
objs=""
for o in build/fpc/*.o; do
  b=$(basename $o .o)
  s=${b%_p[0-9]}; part=""   # kernels_1d_pN.o = kernels_1d.cu compiled with -DFPC_1D_PART=N (build.py)
  [[ $b != $s ]] && part="-DFPC_1D_PART=${b##*_p}"
  if [[ " $srcs " == *" $s "* ]]; then
    nvcc $F $part -c paper_2003_07020_b200/csrc/$s.cu -o build/var_$name/$b.o &
    objs="$objs build/var_$name/$b.o"
  else
    objs="$objs $o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/_timing/$name.so $objs
echo scripts/_timing/$name.so
