#!/bin/bash
# Dev experiment: c2 GEMM stage time vs raw-ring depth / U-ring depth / kc (dbg 0 and 7).
g() { python bench.py --steps 10 --warmup 3 --config ${CFG:-c2} --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['gemm']['ms'])"; }
for d in 0 7; do
  for nr in 2 4 6 8; do echo -n "dbg=$d nraw<=$nr: "; WINO_GEMM_DBG=$d WINO_GEMM_NRAW=$nr g; done
  for nb in 1 2 3; do echo -n "dbg=$d nbr=$nb: "; WINO_GEMM_DBG=$d WINO_GEMM_NBR=$nb g; done
  for kc in 16; do echo -n "dbg=$d kc=$kc: "; WINO_GEMM_DBG=$d WINO_GEMM_KC=$kc g; done
done
