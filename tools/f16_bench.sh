#!/bin/bash
# 3xTF32 vs 3xFP16 (WINO_GEMM_AUTO_MODE) per config, interleaved
for rep in 1 2; do
for mode in 3 4; do
  WINO_GEMM_AUTO_MODE=$mode WINO_FOLD=0 timeout 300 python bench.py --config c4 --extra c2,c3 --steps 30 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/tmp/k.err || tail -3 /tmp/k.err
  python -c "
import json; d=json.load(open('/tmp/k.json'))
for n,c in d['configs'].items(): print('mode=$mode', n, c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))"
done
done
