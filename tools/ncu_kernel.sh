#!/bin/bash
# ncu --set full of one kernel (regex $1) of config $2, exported as raw + source CSV into gpurun_out/$3_*.
# usage: bash tools/ncu_kernel.sh k_input_xform c4 tag [extra env assignments...]
K=$1; C=$2; T=$3; shift 3
mkdir -p gpurun_out
env "$@" timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:$K -s 2 -c 1 -o /tmp/$T \
  python bench.py --steps 2 --warmup 3 --config $C --extra "" --no-cpu-baseline > /tmp/$T.log 2>&1; echo ncu=$?
ncu -i /tmp/$T.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv
ncu -i /tmp/$T.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_source.csv
ncu -i /tmp/$T.ncu-rep --page details --csv > gpurun_out/${T}_details.csv
