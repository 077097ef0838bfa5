#!/bin/bash
g() { python bench.py --steps 10 --warmup 3 --config $1 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['input_xform']['ms'])"; }
for c in ${1:-c4 c2}; do for t in ${2:-256 224 192}; do echo -n "$c threads=$t: "; WINO_IN_THREADS=$t g $c; done; done
