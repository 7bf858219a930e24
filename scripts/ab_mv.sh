#!/bin/bash
# A/B of library variants (scripts/_timing/<name>.so) on the config-1 operator timings (under gpurun)
for v in "$@"; do
  echo "== $v"; FPC_LIB=scripts/_timing/$v.so timeout 200 python scripts/order_timing.py 2>&1 | grep -v Warn | head -1
done
