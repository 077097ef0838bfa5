#!/bin/bash
# dfold tests + c3 A/B (WINO_DFOLD=1 vs 0), interleaved
python -m pytest tests/test_gpu_dfold.py -x -q -s 2>&1 | tail -${TAILN:-25} > gpurun_out/dfold_test.txt
for rep in 1 2; do for d in 1 0; do WINO_DFOLD=$d python bench.py --config c3 --extra "" --steps 20 --warmup 5 --nets "" --nd "" --no-cpu-baseline --no-tf32-peak 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for n,c in d['configs'].items(): print('dfold=$d', n, c['ms_per_layer'], {s:round(v['ms'],4) for s,v in c['stages'].items()}, 'fold_mode', c['info']['fold_mode'])
" >> gpurun_out/dfold_test.txt 2>&1; done; done
cat gpurun_out/dfold_test.txt
