#!/bin/bash
# Dev experiment: input-transform stage time vs slab planning knobs.
g() { python bench.py --steps 10 --warmup 3 --config $1 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['input_xform']['ms'])"; }
for c in c2 c4 c5 c3; do
  echo -n "$c default: "; g $c
  echo -n "$c slots2: "; WINO_IN_SLOTS=2 g $c
  for t in 32 48 128; do echo -n "$c target=${t}KB: "; WINO_IN_TARGET_KB=$t g $c; done
done
