set -u
o=gpurun_out/${1:-d2c4}
mkdir -p $o
export HSW_D2=1
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -m gpu -k "c4 and not full" > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
timeout 600 python tools/quick_bench.py c4 > $o/qb.log 2>&1; echo "rc=$?" >> $o/qb.log
