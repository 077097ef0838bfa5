#!/bin/bash
# a2 in-place H mode: line-aligned phase-2 items (WINO_IN_ALIGN) vs the default, interleaved
g() { python bench.py --steps 20 --warmup 5 --config $1 --extra "" --nets "" --nd "" --no-cpu-baseline --no-tf32-peak 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print(' '.join('%s=%.4f'%(k,v['ms']) for k,v in s.items()), 'ms_per_layer=%.4f'%d['ms_per_step'], 'relL2', (d.get('parity') or {}).get('$1', {}).get('relL2'))"; }
for r in 1 2 3; do for c in ${CFGS:-c4}; do for v in ${VALS:-0 1}; do echo -n "$c align=$v: "; WINO_IN_ALIGN=$v bash -c "$(declare -f g); g $c"; done; done; done
