#!/bin/bash
g() { python bench.py --steps 10 --warmup 3 --config $1 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); s=d['stages']; print(' '.join('%s=%.4f'%(k,v['ms']) for k,v in s.items()))"; }
for c in c2 c5; do for d in 29 31 27; do echo -n "$c dbg=$d: "; WINO_GEMM_DBG=$d WINO_GEMM_VARIANT=1 g $c; done; done
