#!/bin/bash
# PDL per stage (WINO_PDL_MASK: 1 input, 2 GEMM, 4 output transform launched with PDL)
mkdir -p gpurun_out
for rep in 1 2; do for v in 7 3; do
  WINO_PDL_MASK=$v timeout 300 python bench.py --config c4 --extra "c3,c2,c5" --steps 20 --warmup 5 --nets "fig4_f54" --nd "c3t,c3s133,c3t311" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/pdl.json 2> gpurun_out/pdl.err
  python -c "
import json; d=json.load(open('gpurun_out/pdl.json'))
for n,c in d['configs'].items(): print('mask=$v', n, c['ms_per_layer'])
for n,c in d['per_axis_workloads'].items(): print('mask=$v', n, c['ms_per_layer'])
for n,c in d['paper_workloads'].items(): print('mask=$v', n, {b: v['ms_per_pass'] for b, v in c['by_batch'].items()})"
done; done
