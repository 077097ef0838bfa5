#!/bin/bash
# GEMM k-chunk (kc) per variant: stage and step times
for c in ${CFGS:-c2 c3 c4}; do for v in ${VARS:-2 1 0}; do for kc in 32 64; do
  echo -n "$c var=$v kc=$kc: "
  WINO_GEMM_VARIANT=$v WINO_GEMM_BN=128 WINO_GEMM_KC=$kc python bench.py --steps 20 --warmup 3 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'], d['ms_per_step'])"
done; done; done
