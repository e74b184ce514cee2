set -u
o=gpurun_out/${1:-r2b}
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $o/gputests.log 2>&1; echo "rc=$?" >> $o/gputests.log
timeout 300 python __graft_entry__.py --smoke > $o/smoke.log 2>&1; echo "rc=$?" >> $o/smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu > $o/bench.log 2>&1; echo "rc=$?" >> $o/bench.log
