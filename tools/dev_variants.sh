#!/bin/bash
# Development: parity subset + C4 timing + phase profile for each value of an env variable.
# Usage (via gpurun): bash tools/dev_variants.sh VAR "v1 v2 ..." [config]
set -u
name=$1; vals=$2; cfg=${3:-c4}
mkdir -p gpurun_out
for v in $vals; do
  export $name=$v
  echo "=== $name=$v"
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "all_ordinate and $cfg or single_hex or singular_block_3d" 2>&1 | tail -1
  timeout 200 python tools/quick_bench.py $cfg 2>&1 | tail -1
  QUICK=1 timeout 200 python tools/ablate.py $cfg 2>&1 | tail -2
done
