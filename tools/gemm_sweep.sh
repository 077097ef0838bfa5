#!/bin/bash
# GEMM stage time per forced variant / k-chunk (c2 by default)
for c in ${CFGS:-c2}; do for v in 0 1 2; do for kc in 16 32; do
  echo -n "$c var=$v kc=$kc: "
  WINO_GEMM_VARIANT=$v WINO_GEMM_KC=$kc python bench.py --steps 20 --warmup 3 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'], d['ms_per_step'])"
done; done; done
