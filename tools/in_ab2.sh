#!/bin/bash
# A/B of the input-kernel dev flags (WINO_IN_FLAGS) on c4 / c3 / c2 / c5, interleaved
for rep in 1 2 3; do
for f in 0 3; do
  WINO_IN_FLAGS=$f timeout 300 python bench.py --config c4 --extra c3,c2,c5 --steps 30 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/k.json')); print('flags=$f', ' '.join('%s:%.4f'%(n,c['stages']['input_xform']['ms']) for n,c in d['configs'].items()))"
done
done
