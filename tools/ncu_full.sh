# one-level --set full capture of the C4 production kernel + raw/source pages (usage: bash tools/ncu_full.sh TAG [regex])
set -u
tag=${1:-x}; kre=${2:-dmma1}
o=gpurun_out/$tag
mkdir -p $o
HSW_DATAFLOW=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 300 -c 1 \
    -o $o/prof_c4 python tools/profile_case.py c4 32 8 32 2 > $o/ncu_full.log 2>&1
ncu -i $o/prof_c4.ncu-rep --page raw --csv > $o/raw.csv 2>&1
ncu -i $o/prof_c4.ncu-rep --page source --csv --print-source sass > $o/src.csv 2>&1
ncu -i $o/prof_c4.ncu-rep --page details --csv > $o/details.csv 2>&1
rm -f $o/prof_c4.ncu-rep
