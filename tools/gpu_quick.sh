#!/bin/bash
# GPU round trip used during development: gpu tests (stop at first failure) then the bench (no CPU baseline).
mkdir -p gpurun_out
timeout 420 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench.json"))
for n,c in d["configs"].items():
    print(n, c["ms_per_layer"], c["tflops_direct_equiv"], " ".join("%s=%.4f"%(s,v["ms"]) for s,v in c["stages"].items()), "sum=%.4f"%sum(v["ms"] for v in c["stages"].values()))
PY
