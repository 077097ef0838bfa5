#!/bin/bash
# fold GEMM skeleton probes (WINO_FOLD_DBG bits; results invalid) on c5 F=2 and c3 F=1
for cfg in "c5 2" "c3 1"; do
  set -- $cfg
  for dbg in 0 1 2 4 8 16 24 31; do
    WINO_FOLD=$2 WINO_FOLD_RES=0 WINO_FOLD_DBG=$dbg timeout 300 python bench.py --config $1 --extra "" --steps 10 --warmup 3 \
      --nets "" --nd "" --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/k.json')); c=d['configs']['$1']; print('$1 F=$2 dbg=$dbg gemm=%.4f'%c['stages']['gemm']['ms'])"
  done
done
