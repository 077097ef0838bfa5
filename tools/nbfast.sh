#!/bin/bash
for rep in 1 2; do
for nbf in 0 1; do
for mode in 3 4; do
  WINO_GEMM_NBFAST=$nbf WINO_GEMM_AUTO_MODE=$mode WINO_GEMM_VARIANT=2 WINO_FOLD=0 timeout 300 python bench.py --config c4 --extra c2 --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/tmp/k.err || tail -3 /tmp/k.err
  python -c "
import json; d=json.load(open('/tmp/k.json'))
print('nbfast=$nbf mode=$mode', ' '.join('%s %.4f gemm=%.4f'%(n, c['ms_per_layer'], c['stages']['gemm']['ms']) for n,c in d['configs'].items()))"
done; done; done
