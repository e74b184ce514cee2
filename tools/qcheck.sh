# quick GPU check: parity subset + per-config sweep timing (usage: bash tools/qcheck.sh TAG [configs...])
set -u
tag=${1:-q}; shift
o=gpurun_out/$tag
mkdir -p $o
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "all_ordinate or single_hex or local_solve or singular" tests/test_golden.py tests/test_reference_pin.py -m gpu > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
timeout 900 python tools/quick_bench.py ${@:-c4} > $o/qb.log 2>&1; echo "rc=$?" >> $o/qb.log
