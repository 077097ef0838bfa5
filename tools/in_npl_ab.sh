#!/bin/bash
# c4 a2 with line-aligned items: four slabs x 448 threads (plan default) vs two slabs x 256 threads, interleaved
g() { python bench.py --steps 30 --warmup 5 --config c4 --extra "" --nets "" --nd "" --no-cpu-baseline --no-tf32-peak 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print(' '.join('%s=%.4f'%(k,v['ms']) for k,v in s.items()), 'ms_per_layer=%.4f'%d['ms_per_step'])"; }
for r in 1 2 3; do
  echo -n "default (npl 4 x 448): "; bash -c "$(declare -f g); g"
  echo -n "npl 2 x 256:           "; WINO_IN_NPL=2 WINO_IN_THREADS=256 bash -c "$(declare -f g); g"
done
