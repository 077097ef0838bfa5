#!/bin/bash
# Dev experiment: GEMM stage time per schedule (TS/SS, U resident/streamed).
for c in ${1:-c2 c3}; do
  for ts in 1 0; do for res in 1 0; do
    echo -n "$c ts=$ts res=$res: "
    WINO_GEMM_TS=$ts WINO_GEMM_RES=$res python bench.py --steps 10 --warmup 3 --config $c --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"
  done; done
done
