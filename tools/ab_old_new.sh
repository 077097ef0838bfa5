b() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --extra "c4" 2>/dev/null | python -c "
import json,sys
d=json.load(sys.stdin)
for n,c in d['configs'].items(): print(n, c['ms_per_layer'], ' '.join('%s=%.4f'%(s,v['ms']) for s,v in c['stages'].items()))"; }
echo new; b; cp paper_1611_06565_b200/libwino.so /tmp/new.so; cp _old/libwino.so paper_1611_06565_b200/libwino.so; echo old; b; cp /tmp/new.so paper_1611_06565_b200/libwino.so; echo new; b
