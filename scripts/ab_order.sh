#!/bin/bash
# A/B of library variants (scripts/_timing/<name>.so): config-1 PC apply + solve, both PC orderings (under gpurun)
for v in "$@"; do
  echo "== $v"; FPC_LIB=scripts/_timing/$v.so timeout 200 python scripts/order_timing.py 2>&1 | grep -v Warn | cut -c1-330
done
