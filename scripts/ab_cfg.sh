#!/bin/bash
# A/B of library variants (scripts/_timing/<name>.so) on scripts/cfg_timing.py; usage: ab_cfg.sh "<configs>" v1 v2 ...
cfgs=$1; shift
for v in "$@"; do
  echo "== $v"; FPC_LIB=scripts/_timing/$v.so timeout 300 python scripts/cfg_timing.py $cfgs 2>&1 | grep -v Warn
done
