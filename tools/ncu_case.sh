# --set full capture of one level of a config's sweep kernel (usage: bash tools/ncu_case.sh TAG CFG KREGEX SKIP [env...])
set -u
tag=$1; cfg=$2; kre=$3; skip=$4
o=gpurun_out/$tag
mkdir -p $o
case $cfg in c5) args="c5 24 8 32 2";; c4) args="c4 32 8 32 2";; *) args="$cfg";; esac
HSW_DATAFLOW=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 \
    -o $o/prof python tools/profile_case.py $args > $o/ncu_full.log 2>&1
ncu -i $o/prof.ncu-rep --page raw --csv > $o/raw.csv 2>&1
ncu -i $o/prof.ncu-rep --page source --csv --print-source sass > $o/src.csv 2>&1
rm -f $o/prof.ncu-rep
