#!/bin/bash
# e2e (host-buffer forward) time vs chunk count and ramp, per config
for c in ${CFGS:-c2 c5}; do for r in 0 1; do for n in ${NCHS:-4 6 8 12 16}; do
echo -n "$c ramp=$r nch=$n: "; WINO_HOST_RAMP=$r WINO_HOST_CHUNKS=$n python bench.py --steps 10 --warmup 3 --config $c --extra "" --nets "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['e2e']['ms_per_step'])"
done; done; done
