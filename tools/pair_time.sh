#!/bin/bash
# Dev experiment: GEMM stage time, CTA pair on/off.
for c in ${1:-c2 c3}; do for p in 0 1 2; do
  echo -n "$c variant=$p: "; WINO_GEMM_VARIANT=$p python bench.py --steps 10 --warmup 3 --config $c --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"
done; done
