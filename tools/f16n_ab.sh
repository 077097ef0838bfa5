#!/bin/bash
# GPU check of the V-resident 3xFP16 GEMM (k_gemm_f16n) and the filter-side fold:
# new parity tests, then A/B bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ufold.py tests/test_gpu_f16.py -q -x --timeout 600 > gpurun_out/t_ufold.log 2>&1; echo pytest=$?; tail -3 gpurun_out/t_ufold.log
run() {  # tag, configs, env...
  local tag=$1 cfgs=$2; shift 2
  local first=${cfgs%%,*} rest=${cfgs#*,}
  [ "$rest" = "$cfgs" ] && rest=""
  env "$@" timeout 300 python bench.py --config $first --extra "$rest" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err || { echo "$tag failed"; tail -5 gpurun_out/ab_$tag.err; return; }
  python - $tag <<'PY'
import json, sys
t = sys.argv[1]
d = json.load(open("gpurun_out/ab_%s.json" % t))
for n, c in d["configs"].items():
    print("%-8s %s %.4f ms  fold=%s/%s gemm=%s |" % (t, n, c["ms_per_layer"], c["info"].get("fold"),
          c["info"].get("fold_mode"), c.get("gemm_scheme")),
          " ".join("%s=%.4f" % (s, v["ms"]) for s, v in c["stages"].items()))
PY
}
for rep in 1 2; do
run c4new$rep c4
run c4old$rep c4 WINO_F16N=0
done
run c3uf1 c3 WINO_UFOLD=1
run c3uf1noskip c3 WINO_UFOLD=1 WINO_UFOLD_SKIP=0
run c3uf1old c3 WINO_UFOLD=1 WINO_F16N=0
run c5uf2 c5 WINO_UFOLD=2
