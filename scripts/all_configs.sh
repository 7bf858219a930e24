#!/bin/bash
# One bench line per BASELINE config on one B200 (run under gpurun): configs 0, 1 (both gammas,
# both PC orderings), 2 and 3.  usage: bash scripts/all_configs.sh <tag>
set -u
tag=${1:-r1}
mkdir -p gpurun_out
out=gpurun_out/${tag}_configs.jsonl
: > $out
run() { timeout ${T:-600} python bench.py "$@" >> $out 2>> gpurun_out/${tag}_configs.err || echo "{\"failed\": \"$*\"}" >> $out; }
run --config 0
run --config 1 --gamma 1.2
run --config 1 --gamma 1.2 --ordering commuted --no-cpu-baseline
run --config 1 --gamma 1.8
run --config 2
T=1500 run --config 3 --steps 2 --warmup 3
wc -l $out
