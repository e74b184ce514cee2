#!/bin/bash
# Round-end measurement batch on the GPU box (one GPU): tests, bench line, reference arm,
# per-config report, ncu launch list, whole-sweep DRAM traffic, one-level full capture.
# Usage (via gpurun): bash tools/round_measure.sh TAG
set -u
tag=${1:-r1}
o=gpurun_out/$tag
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/gputests.log 2>&1; echo "rc=$?" >> $o/gputests.log
timeout 600 python bench.py --steps 5 --warmup 3 > $o/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.log 2>&1
timeout 900 python tools/report_configs.py $o/configs.md > $o/configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches.csv \
    python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e > $o/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
    --clock-control none -k regex:dmma1 -c 1 --csv --log-file $o/traffic.csv python tools/profile_case.py c4 32 8 32 1 > $o/ncu_traffic.log 2>&1
HSW_DATAFLOW=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma1 -s 300 -c 1 \
    -o $o/prof_c4 python tools/profile_case.py c4 32 8 32 2 > $o/ncu_full.log 2>&1
ncu -i $o/prof_c4.ncu-rep --page raw --csv > $o/raw.csv 2>&1
ncu -i $o/prof_c4.ncu-rep --page source --csv --print-source sass > $o/src.csv 2>&1
rm -f $o/prof_c4.ncu-rep
