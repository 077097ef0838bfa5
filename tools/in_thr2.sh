#!/bin/bash
# c4 input-transform block size (four-slab in-place H mode): phase-2 round quantisation
mkdir -p gpurun_out
for rep in 1 2; do
for t in 384 416 448 512; do
  WINO_IN_THREADS=$t timeout 300 python bench.py --config c4 --extra "" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/thr_$t.json 2> gpurun_out/thr_$t.err
  python -c "
import json; d=json.load(open('gpurun_out/thr_$t.json')); c=d['configs']['c4']
print('thr=$t', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))"
done
done
