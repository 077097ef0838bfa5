#!/bin/bash
# a2 L2 slab prefetch distance sweep (WINO_IN_PREFETCH = CTAs ahead): stage times per config
g() { python bench.py --steps 20 --warmup 5 --config $1 --extra "" --nets "" --nd "" --no-cpu-baseline --no-tf32-peak 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print(' '.join('%s=%.4f'%(k,v['ms']) for k,v in s.items()), 'ms_per_layer=%.4f'%d['ms_per_step'])"; }
for r in 1 2; do for c in ${CFGS:-c4 c2 c3 c5}; do for v in ${VALS:-0 148 296 592}; do echo -n "$c prefetch=$v: "; WINO_IN_PREFETCH=$v bash -c "$(declare -f g); g $c"; done; done; done
