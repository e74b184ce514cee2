#!/bin/bash
# Development loop on the GPU box: quick parity subset + C4 timing + phase profile.
# Usage (via gpurun): bash tools/dev_check.sh [configs...]
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "all_ordinate or single_hex or singular_block_3d or full_config_sampled" > gpurun_out/dev_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/dev_tests.log
tail -3 gpurun_out/dev_tests.log
timeout 300 python tools/quick_bench.py ${@:-c4} > gpurun_out/dev_bench.log 2>&1; cat gpurun_out/dev_bench.log
QUICK=1 timeout 300 python tools/ablate.py c4 > gpurun_out/dev_ablate.log 2>&1; cat gpurun_out/dev_ablate.log
