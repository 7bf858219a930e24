#!/bin/bash
# config 0 and config 1 solve times with the in-tree library (under gpurun)
python bench.py --config 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg0', round(d['ms_per_step'],3), d['iterations'], {k: round(v,3) for k,v in d['kernel_time_ms_per_solve'].items()})"
python scripts/order_timing.py 2>&1 | grep -v Warn | cut -c1-330
