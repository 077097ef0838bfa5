#!/bin/bash
# L2-chunked pipeline (fuse=4) vs unfused, per config and chunk size (MB of V + M per chunk)
for c in ${CFGS:-c2 c3 c5}; do
  echo -n "$c unfused: "; python bench.py --steps 20 --warmup 3 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'])"
  for mb in ${MBS:-24 48 96}; do
    echo -n "$c fuse=4 chunk=${mb}MB: "; WINO_CHUNK_MB=$mb python bench.py --steps 20 --warmup 3 --fuse 4 --config $c --extra "" --nets "" --nd "" --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['configs'][list(d['configs'])[0]]['info']['chunk_slabs'])"
  done
done
