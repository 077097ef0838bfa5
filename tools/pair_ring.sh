#!/bin/bash
# CTA-pair GEMM: U ring depth (nbr) vs raw V ring depth (nraw), stage and step times
for c in ${CFGS:-c2 c3}; do for nb in 4 6 8; do for nr in 8 6 4; do
  echo -n "$c nbr=$nb nraw=$nr: "
  WINO_GEMM_VARIANT=2 WINO_GEMM_BN=128 WINO_GEMM_NBR=$nb WINO_GEMM_NRAW=$nr python bench.py --steps 20 --warmup 3 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'], d['ms_per_step'])"
done; done; done
