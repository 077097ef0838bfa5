#!/bin/bash
# fold GEMM knob sweep on c5 (F=2) and c3 (F=1): A stages, U residency
mkdir -p gpurun_out
for cfg in "c5 2" "c3 1"; do
  set -- $cfg
  for na in 2 4 6 8; do
    for res in 0 1; do
      WINO_FOLD=$2 WINO_FOLD_NA=$na WINO_FOLD_RES=$res timeout 300 python bench.py --config $1 --extra "" --steps 20 --warmup 5 \
        --nets "" --nd "" --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/dev/null
      python -c "import json; d=json.load(open('/tmp/k.json')); c=d['configs']['$1']; print('$1 F=$2 na=$na res=$res', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))"
    done
  done
done
