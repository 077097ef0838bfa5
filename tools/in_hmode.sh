#!/bin/bash
g() { python bench.py --steps 10 --warmup 3 --config c4 --extra "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['stages']['input_xform']['ms'], d['configs']['c4']['info']['in_slab_tiles'])"; }
for t in 24 48; do echo -n "c4 H target=${t}KB: "; WINO_IN_TARGET_KB=$t g; done
