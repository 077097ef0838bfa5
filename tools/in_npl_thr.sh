#!/bin/bash
# c4 a2 sweep: slabs per CTA x block size (input-transform stage time, step time)
g() { python bench.py --steps 10 --warmup 3 --config ${CFG:-c4} --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('input=%.4f'%s['input_xform']['ms'], 'step=%.4f'%d['ms_per_step'])"; }
for n in ${NPLS:-2 3 4 6 8}; do for t in ${THRS:-256 384 512}; do echo -n "npl=$n thr=$t: "; WINO_IN_NPL=$n WINO_IN_THREADS=$t bash -c "$(declare -f g); g"; done; done
