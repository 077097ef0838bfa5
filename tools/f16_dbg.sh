#!/bin/bash
for d in 0 1 2 4 3 7; do
  WINO_F16_DBG=$d WINO_GEMM_AUTO_MODE=4 WINO_FOLD=0 timeout 300 python bench.py --config c4 --extra c2 --steps 10 --warmup 3 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/tmp/k.err || tail -3 /tmp/k.err
  python -c "
import json; d=json.load(open('/tmp/k.json'))
print('dbg=$d', ' '.join('%s gemm=%.4f'%(n, c['stages']['gemm']['ms']) for n,c in d['configs'].items()))"
done
