#!/bin/bash
# c4 input transform probe: time without V stores (WINO_IN_FLAGS=4, results invalid)
mkdir -p gpurun_out
for tag in base nostore base2 nostore2; do
  case $tag in nostore*) E="WINO_IN_FLAGS=4";; *) E="WINO_IN_FLAGS=0";; esac
  env $E timeout 300 python bench.py --config c4 --extra "" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/pr_$tag.json 2> gpurun_out/pr_$tag.err
  python -c "
import json; d=json.load(open('gpurun_out/pr_$tag.json')); c=d['configs']['c4']
print('%-10s'%'$tag', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))" 2>&1 | tail -1
done
