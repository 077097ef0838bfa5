#!/bin/bash
# Dev experiment: MMA chain alone (dbg 27 = no loads, no conversion, no stores) per variant / config.
g() { python bench.py --steps 10 --warmup 3 --config $1 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print('gemm=%.4f'%s['gemm']['ms'])"; }
for c in c2 c4 c5; do for v in 0 1 2; do for d in 27 31; do echo -n "$c variant=$v dbg=$d: "; WINO_GEMM_DBG=$d WINO_GEMM_VARIANT=$v g $c; done; done; done
