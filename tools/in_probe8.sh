#!/bin/bash
# c4 input transform probes (results invalid): WINO_IN_FLAGS=8 staging only, =4 no V stores
mkdir -p gpurun_out
for tag in base stage nostore base2 stage2 nostore2; do
  case $tag in stage*) E="WINO_IN_FLAGS=8";; nostore*) E="WINO_IN_FLAGS=4";; *) E="WINO_IN_FLAGS=0";; esac
  for thr in 416 448; do
  env $E WINO_IN_THREADS=$thr timeout 300 python bench.py --config c4 --extra "" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/pr_$tag.json 2> gpurun_out/pr_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/pr_$tag.json')); c=d['configs']['c4']
print('%-10s thr=$thr'%'$tag', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))" 2>&1 | tail -1
  done
done
