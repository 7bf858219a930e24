#!/bin/bash
# Bench line + ncu launch list + one `ncu --set full` capture per hot kernel (run under gpurun).
# usage: bash scripts/profile_round.sh <tag>
set -u
tag=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || { echo "bench failed"; tail -20 gpurun_out/${tag}_bench.err; exit 1; }
tail -c 400 gpurun_out/${tag}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_list.log 2>&1 || echo "launch list failed"
ncu --set full --clock-control none --import-source on \
  -k regex:"k_matvec_split|k_tau_solve_1d|k_time_fwd|k_time_inv|k_dots2|k_update2|k_dots|k_update" \
  --launch-skip 14 -c 7 -o gpurun_out/${tag}_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1 || echo "full capture failed"
ls -la gpurun_out/ | grep ${tag}
