#!/bin/bash
# Development loop for the static-pivot kernel: parity subset, timings with and without it.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "all_ordinate or single_hex or singular_block or full_config_sampled" > gpurun_out/sp_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/sp_tests.log
tail -15 gpurun_out/sp_tests.log
timeout 600 python tools/quick_bench.py ${@:-c1 c2 c3 c4} > gpurun_out/sp_bench.log 2>&1; cat gpurun_out/sp_bench.log
HSW_SP_Q4=1 timeout 600 python tools/quick_bench.py c5 > gpurun_out/sp_bench_c5.log 2>&1; cat gpurun_out/sp_bench_c5.log
