#!/bin/bash
# Alternating A/B of an env knob on step time and stages: KNOB=X A=0 B=1 CFGS="c2 c3" REPS=3 bash tools/ab_env.sh
g() { python bench.py --steps ${STEPS:-30} --warmup 5 --config $1 --extra "" --nets "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('step=%.4f'%d['ms_per_step'], ' '.join('%s=%.4f'%(k[:3],v['ms']) for k,v in s.items()))"; }
for c in ${CFGS:-c2}; do for r in $(seq ${REPS:-3}); do for v in ${A:-0} ${B:-1}; do echo -n "$c $KNOB=$v: "; env $KNOB=$v bash -c "$(declare -f g); g $c"; done; done; done
