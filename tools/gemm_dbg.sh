#!/bin/bash
# Dev experiment: GEMM stage time of one forced variant under WINO_GEMM_DBG knobs
# (results invalid when != 0).  usage: VAR=2 CFGS="c2 c5" DBGS="0 1 8 16" bash tools/gemm_dbg.sh
for c in ${CFGS:-c2}; do
  for d in ${DBGS:-0 1}; do
    echo -n "$c var=${VAR:-2} dbg=$d: "
    WINO_GEMM_VARIANT=${VAR:-2} WINO_GEMM_DBG=$d python bench.py --steps 10 --warmup 3 --config $c --extra "" --nets "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"
  done
done
