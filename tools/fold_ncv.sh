#!/bin/bash
for ncv in 4 8; do
  for cfg in "c5 2" "c3 1" "c3 2"; do
    set -- $cfg
    WINO_FOLD=$2 WINO_FOLD_NCV=$ncv timeout 300 python bench.py --config $1 --extra "" --steps 20 --warmup 5 \
      --nets "" --nd "" --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/k.json')); c=d['configs']['$1']; print('ncv=$ncv $1 F=$2', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))"
  done
done
