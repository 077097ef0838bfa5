#!/bin/bash
# A/B of the in-tree libwino.so against _old/libwino.so (an older build) on the same box.
# usage: CFGS="c3 c4" bash tools/ab_old_new.sh
b() { for c in ${CFGS:-c2 c4}; do echo -n "$1 $c: "; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $c --extra "" --nets "" 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
for n,c in d['configs'].items(): print(c['ms_per_layer'], ' '.join('%s=%.4f'%(s,v['ms']) for s,v in c['stages'].items()))"; done; }
cp paper_1611_06565_b200/libwino.so /tmp/new.so
b new; cp _old/libwino.so paper_1611_06565_b200/libwino.so; b old; cp /tmp/new.so paper_1611_06565_b200/libwino.so; b new; cp _old/libwino.so paper_1611_06565_b200/libwino.so; b old; cp /tmp/new.so paper_1611_06565_b200/libwino.so
