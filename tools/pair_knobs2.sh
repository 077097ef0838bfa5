#!/bin/bash
for v in 1 2; do for d in 5 13 21 29; do
  echo -n "c2 variant=$v dbg=$d: "; WINO_GEMM_DBG=$d WINO_GEMM_VARIANT=$v python bench.py --steps 10 --warmup 3 --config c2 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"
done; done
