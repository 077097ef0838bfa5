#!/bin/bash
# CTA-pair GEMM unit order: xi-major (0) vs m-pair-major (1)
for c in ${CFGS:-c2 c3 c4}; do for r in 1 2; do for o in 0 1; do
  echo -n "$c order=$o: "
  WINO_GEMM_VARIANT=2 WINO_GEMM_BN=128 WINO_GEMM_ORDER=$o python bench.py --steps 20 --warmup 3 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'], d['ms_per_step'])"
done; done; done
