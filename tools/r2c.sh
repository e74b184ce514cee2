set -u
o=gpurun_out/r2c
mkdir -p $o
./tools/dmma_check/tmem_rate > $o/tmem_rate.log 2>&1
./tools/dmma_check/dmma_rate > $o/dmma_rate.log 2>&1
FLAGS=0,256,320,257,258,260 ONLY_FLAGS=1 timeout 600 python tools/ablate.py c4 > $o/ablate_c4.log 2>&1
