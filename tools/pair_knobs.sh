#!/bin/bash
for p in 1 0; do for d in 0 1 4 5; do
  echo -n "c2 pair=$p dbg=$d: "; WINO_GEMM_DBG=$d WINO_GEMM_PAIR=$p python bench.py --steps 10 --warmup 3 --config c2 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"
done; done
