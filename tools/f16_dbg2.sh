#!/bin/bash
for env in "WINO_L2_HINTS=1" "WINO_L2_HINTS=0"; do
  env $env WINO_GEMM_AUTO_MODE=4 WINO_FOLD=0 timeout 300 python bench.py --config c3 --extra c4 --steps 10 --warmup 3 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/tmp/k.err || tail -3 /tmp/k.err
  python -c "
import json; d=json.load(open('/tmp/k.json'))
print('$env f16', ' '.join('%s gemm=%.4f'%(n, c['stages']['gemm']['ms']) for n,c in d['configs'].items()))"
  env $env WINO_GEMM_AUTO_MODE=3 WINO_FOLD=0 timeout 300 python bench.py --config c3 --extra c4 --steps 10 --warmup 3 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/tmp/k.err || tail -3 /tmp/k.err
  python -c "
import json; d=json.load(open('/tmp/k.json'))
print('$env tf32', ' '.join('%s gemm=%.4f'%(n, c['stages']['gemm']['ms']) for n,c in d['configs'].items()))"
done
