#!/bin/bash
# Development loop for the left-looking static-pivot LU: parity subset, timings with and without it.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "all_ordinate or single_hex or singular_block or full_config_sampled" > gpurun_out/ll_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ll_tests.log
tail -15 gpurun_out/ll_tests.log
timeout 600 python tools/quick_bench.py ${@:-c3 c4} > gpurun_out/ll_bench.log 2>&1; cat gpurun_out/ll_bench.log
HSW_LL=0 timeout 600 python tools/quick_bench.py ${@:-c3 c4} > gpurun_out/ll_bench_rl.log 2>&1; cat gpurun_out/ll_bench_rl.log
