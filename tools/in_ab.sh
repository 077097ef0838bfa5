#!/bin/bash
# A/B of an input-transform env knob: stage times of the input transform per config.
# usage: KNOB=WINO_IN_HINPLACE VALS="0 1" CFGS="c4 c2" bash tools/in_ab.sh
g() { python bench.py --steps 10 --warmup 3 --config $1 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print(' '.join('%s=%.4f'%(k,v['ms']) for k,v in s.items()), 'ms_per_layer=%.4f'%d['ms_per_step'])"; }
for c in ${CFGS:-c4 c2}; do for v in ${VALS:-0 1}; do echo -n "$c $KNOB=$v: "; env $KNOB=$v bash -c "$(declare -f g); g $c"; done; done
