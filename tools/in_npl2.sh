#!/bin/bash
# c4 input transform: slabs per CTA x block size (in-place H mode, pad8 item slots)
mkdir -p gpurun_out
one() {
  WINO_IN_NPL=$1 WINO_IN_THREADS=$2 timeout 300 python bench.py --config c4 --extra "" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/np.json 2> gpurun_out/np.err || { echo "npl=$1 thr=$2 failed"; return; }
  python -c "
import json; d=json.load(open('gpurun_out/np.json')); c=d['configs']['c4']
print('npl=$1 thr=$2', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))"
}
for rep in 1 2; do
one 4 448
one 2 224
one 2 256
one 2 352
one 3 256
one 3 352
one 1 224
done
