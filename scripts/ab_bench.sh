#!/bin/bash
# usage: scripts/ab_bench.sh name1 name2 ...  (name "default" = the in-tree library)
for n in "$@"; do
  if [ "$n" = default ]; then unset FPC_LIB; else export FPC_LIB=scripts/_timing/$n.so; fi
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$n',round(d['ms_per_step'],3),{a:round(b,3) for a,b in d['kernel_time_ms_per_solve'].items()})"
done
