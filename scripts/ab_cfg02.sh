#!/bin/bash
# A/B of library variants on configs 0 and 2 (solve time + per-kernel live times), under gpurun
for v in "$@"; do
  for c in 0 2; do
    FPC_LIB=scripts/_timing/$v.so python bench.py --config $c --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'cfg$c', round(d['ms_per_step'],3), d['iterations'], {k: round(v*1e3/d['kernel_launches_per_solve'][k],1) for k,v in d['kernel_time_ms_per_solve'].items()})"
  done
done
