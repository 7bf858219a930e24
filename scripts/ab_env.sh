#!/bin/bash
# A/B of library variants x environment settings on scripts/solve_timing.py
# usage: ab_env.sh "<configs>" "<lib1 lib2 ...>" "ENV1=a ENV2=b" "ENV1=c" ...   (use "-" for no env)
cfgs=$1; libs=$2; shift 2
for v in $libs; do
  for e in "$@"; do
    [ "$e" = "-" ] && e=""
    echo "== $v [$e]"
    env $e FPC_LIB=scripts/_timing/$v.so timeout 600 python scripts/solve_timing.py $cfgs 2>&1 | grep -v Warn
  done
done
