#!/bin/bash
# A/B of library variants on one config-3 matvec + PC apply (scripts/op_once.py timing), under gpurun
for v in "$@"; do
  echo "== $v"; FPC_LIB=scripts/_timing/$v.so python scripts/op_timing.py 3
done
