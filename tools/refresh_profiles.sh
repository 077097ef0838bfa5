#!/bin/bash
# Round-end evidence on one GPU (outputs in gpurun_out/, copied to profiles/ by hand):
#   ${T}_pytest_gpu.log   pytest -m gpu
#   ${T}_smoke.log        __graft_entry__.smoke()
#   ${T}_<cfg>_raw.csv    ncu --set full of the three forward kernels of every config, the plan's own choices
#   ${T}_ncu_traffic.json dram read + write bytes per launch from those captures (profiles/ncu_traffic.json),
#                         regenerated BEFORE the bench so the bench line's roofline.traffic is this run's
#   ${T}_bench.json       the default bench line (c4 headline, all configs, cpu_baseline, parity, nets, per-axis)
#   ${T}_reference.json   bench.py --impl reference (the oracle arm)
#   ${T}_launches_c4.csv  ncu launch list (gpu__time_duration) of the headline bench command
# usage: TAG=r02f bash tools/refresh_profiles.sh
T=${TAG:-r02h}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$?
TR=""
for c in c4 c2 c3 c5 c1; do
  timeout 600 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_input|k_gemm|k_output" -s 9 -c 3 -o /tmp/${T}_$c \
    python bench.py --steps 2 --warmup 3 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline --no-tf32-peak \
    > /tmp/${T}_$c.log 2>&1; echo ncu_$c=$?
  ncu -i /tmp/${T}_$c.ncu-rep --page raw --csv > gpurun_out/${T}_${c}_raw.csv
  TR="$TR $c=gpurun_out/${T}_${c}_raw.csv"
done
python tools/ncu_traffic.py $TR > /dev/null && cp profiles/ncu_traffic.json gpurun_out/${T}_ncu_traffic.json; echo traffic=$?
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err; echo reference=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches_c4.csv python bench.py --steps 3 --warmup 3 --extra "" --nets "" --nd "" \
  --no-cpu-baseline --no-tf32-peak > /tmp/${T}_launch.log 2>&1; echo launches=$?
python tools/ncu_summary.py gpurun_out/${T}_c4_raw.csv gpurun_out/${T}_c2_raw.csv gpurun_out/${T}_c3_raw.csv \
  gpurun_out/${T}_c5_raw.csv gpurun_out/${T}_c1_raw.csv > gpurun_out/${T}_ncu_summary.txt 2>&1
