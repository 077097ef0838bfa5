#!/bin/bash
g() { python bench.py --steps 10 --warmup 3 --config ${CFG:-c2} --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['input_xform']['ms'])"; }
for tma in 1 0; do for d in 0 2 3; do echo -n "${CFG:-c2} tma=$tma in_dbg=$d: "; WINO_IN_TMA=$tma WINO_IN_DBG=$d g; done; done
