#!/bin/bash
# Round-end evidence on one GPU: GPU tests, the default bench line, and for
# every config an `ncu --set full` capture of its three kernels (GEMM forced
# to the variant / N tile the bench's plan chose) plus the c2 launch list.
# usage: TAG=r01e bash tools/refresh_profiles.sh   (outputs in gpurun_out/)
T=${TAG:-r01e}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/${T}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench=$?
for c in c2 c3 c4 c5; do
  read V BN <<< $(python -c "import json; d=json.load(open('gpurun_out/${T}_bench.json'))['configs']['$c']['info']; print(d['gemm_variant'], d['n_blk'])")
  echo "$c variant=$V bn=$BN"
  WINO_GEMM_VARIANT=$V WINO_GEMM_BN=$BN timeout 600 ncu -f --set full --import-source on --clock-control none \
    -k regex:"k_input|k_gemm|k_output" -s 9 -c 3 -o /tmp/${T}_$c \
    python bench.py --steps 2 --warmup 3 --config $c --extra "" --nets "" --no-cpu-baseline > /tmp/${T}_$c.log 2>&1; echo ncu_$c=$?
  ncu -i /tmp/${T}_$c.ncu-rep --page raw --csv > gpurun_out/${T}_${c}_raw.csv
done
# the per-axis c3 layer (F(2,3) time x F(4,3)^2 space): its three fused kernels
VT=$(python tools/run_nd.py c3t 1 | awk '{print $3}')
WINO_GEMM_VARIANT=$VT timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"k_input|k_gemm|k_output" -c 3 \
  -o /tmp/${T}_c3t python tools/run_nd.py c3t 3 > /tmp/${T}_c3t.log 2>&1; echo ncu_c3t=$? variant=$VT
ncu -i /tmp/${T}_c3t.ncu-rep --page raw --csv > gpurun_out/${T}_c3t_raw.csv
read V BN <<< $(python -c "import json; d=json.load(open('gpurun_out/${T}_bench.json'))['configs']['c2']['info']; print(d['gemm_variant'], d['n_blk'])")
WINO_GEMM_VARIANT=$V WINO_GEMM_BN=$BN timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches_c2.csv python bench.py --steps 3 --warmup 3 --extra "" --nets "" --no-cpu-baseline \
  > /tmp/${T}_launch.log 2>&1; echo launches=$?
