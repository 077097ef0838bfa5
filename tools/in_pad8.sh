#!/bin/bash
# c4 input transform: pad8 item mapping (conflict-free phase-2 loads) x block size
mkdir -p gpurun_out
one() {  # tag env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --config c4 --extra "" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/p8_$tag.json 2> gpurun_out/p8_$tag.err || { echo "$tag failed"; tail -3 gpurun_out/p8_$tag.err; return; }
  python -c "
import json; d=json.load(open('gpurun_out/p8_$tag.json')); c=d['configs']['c4']
print('%-12s'%'$tag', c['ms_per_layer'], ' '.join('%s=%.4f'%(k,v['ms']) for k,v in c['stages'].items()))"
}
for rep in 1 2; do
one pad8auto
one pad0_416 WINO_IN_PAD8=0 WINO_IN_THREADS=416
one pad8_384 WINO_IN_THREADS=384
one pad8_512 WINO_IN_THREADS=512
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -x -k "c4 or guard or hmode or inplace" > gpurun_out/p8_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/p8_tests.log
