#!/bin/bash
g() { python bench.py --steps 10 --warmup 3 --config c4 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('gemm=%.4f'%d['stages']['gemm']['ms'], d['configs']['c4']['info'])"; }
for bn in 256 128; do for v in 0 1 2; do echo -n "c4 bn=$bn variant=$v: "; WINO_GEMM_BN=$bn WINO_GEMM_VARIANT=$v g; done; done
