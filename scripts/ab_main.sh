#!/bin/bash
# A/B of environment settings on the in-tree library; usage: ab_main.sh "<configs>" "ENV=a" "ENV=b" ... ("-" = none)
cfgs=$1; shift
for e in "$@"; do
  [ "$e" = "-" ] && e=""
  echo "== [$e]"
  env $e timeout 900 python scripts/solve_timing.py $cfgs 2>&1 | grep -v Warn
done
