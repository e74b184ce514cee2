#!/bin/bash
# Round measurement batch on the GPU box (one GPU): tests, bench line (with the per-config
# report), reference arm, ncu launch list, whole-sweep DRAM traffic (C4), one-level --set full
# captures of the C4 (dmma1) and C5 (dmma2) kernels.  Usage (via gpurun): bash tools/round_measure.sh TAG [notests]
set -u
tag=${1:-r2}
o=gpurun_out/$tag
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/smi.txt 2>&1
if [ "${2:-}" != "notests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/gputests.log 2>&1; echo "rc=$?" >> $o/gputests.log
fi
HSW_SETUP_TIMING=1 timeout 900 python bench.py --steps 5 --warmup 3 > $o/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e --skip-per-config > $o/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
    --clock-control none -k regex:dmma1 -c 1 --csv --log-file $o/traffic.csv python tools/profile_case.py c4 32 8 32 1 > $o/ncu_traffic.log 2>&1
bash tools/ncu_case.sh $tag/c4 c4 dmma1 300
bash tools/ncu_case.sh $tag/c5 c5 dmma2 200
