#!/bin/bash
for f in 0 4 0 4; do
  WINO_IN_FLAGS=$f timeout 300 python bench.py --config c4 --extra "" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > /tmp/k.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/k.json')); print('flags=$f', ' '.join('%s:%.4f'%(n,c['stages']['input_xform']['ms']) for n,c in d['configs'].items()))"
done
