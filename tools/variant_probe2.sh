#!/bin/bash
# each (config, variant, resident) in its own process under a timeout
for c in ${1:-c1s c2s c3s c4s c5s}; do for v in 0 1; do for r in 0 1; do
  echo -n "$c v=$v res=$r: "; (WINO_GEMM_RES=$r timeout 60 python tools/variant_probe.py $c $v 2>&1 || echo TIMEOUT) | tail -1
done; done; done
