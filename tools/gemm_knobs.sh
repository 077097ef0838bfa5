#!/bin/bash
# Dev experiment: GEMM stage time under WINO_GEMM_DBG knobs (results invalid when != 0).
for c in ${1:-c2 c3}; do
  for d in 0 1 2 4 3 7; do
    echo -n "$c dbg=$d: "
    WINO_GEMM_DBG=$d python bench.py --steps 10 --warmup 3 --config $c --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"
  done
done
