#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (tools/sanitize_driver.py), once per tcgen05 GEMM variant.  Logs in gpurun_out/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for v in 0 1 2; do
    log=gpurun_out/sanitize_${tool}_v${v}.log
    WINO_GEMM_VARIANT=$v timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_driver.py all > $log 2>&1
    echo "$tool variant=$v rc=$? $(grep -c 'ok$' $log) ok-lines; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK' $log | tail -1)"
  done
done
