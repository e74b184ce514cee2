#!/bin/bash
# A/B of HSW_TUNE / HSW_LL variants on one config (usage: bash tools/tune_check.sh CFG "ENV1" "ENV2" ...)
set -u
cfg=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" | tee -a gpurun_out/tune.log
  env $v timeout 600 python tools/quick_bench.py $cfg 2>&1 | tee -a gpurun_out/tune.log
done
