#!/bin/bash
for c in ${1:-c1s c2s c3s c5s c2}; do for v in 0 1 2; do
  timeout 60 python tools/variant_probe.py $c $v 2>&1 | tail -1 || echo "$c variant $v: TIMEOUT/FAIL"
done; done
