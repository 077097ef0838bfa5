#!/bin/bash
# A/B of the a5 filter-side fold (WINO_UFOLD=F) against the epilogue fold / unfused plans.
mkdir -p gpurun_out
run() {  # tag, configs, env...
  local tag=$1 cfgs=$2; shift 2
  local first=${cfgs%%,*} rest=${cfgs#*,}
  [ "$rest" = "$cfgs" ] && rest=""
  env "$@" timeout 300 python bench.py --config $first --extra "$rest" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/uf_$tag.json 2> gpurun_out/uf_$tag.err || { echo "$tag failed"; tail -5 gpurun_out/uf_$tag.err; return; }
  python - $tag <<'PY'
import json, sys
t = sys.argv[1]
d = json.load(open("gpurun_out/uf_%s.json" % t))
for n, c in d["configs"].items():
    par = d.get("parity", {}).get(n, {})
    print("%-8s %s %.4f ms  fold=%s/%s gemm=%s relL2=%s max=%s pass=%s |" % (t, n, c["ms_per_layer"], c["info"].get("fold"),
          c["info"].get("fold_mode"), c.get("gemm_scheme"), par.get("relL2"), par.get("max_over_maxy"), par.get("pass")),
          " ".join("%s=%.4f" % (s, v["ms"]) for s, v in c["stages"].items()))
PY
}
run base c3,c5,c2
for F in ${UF_LIST:-1 2}; do run "F$F" c3,c5 WINO_UFOLD=$F; done
run c5F3 c5 WINO_UFOLD=3
run c2F1 c2 WINO_UFOLD=1
run c3F1tf c3 WINO_UFOLD=1 WINO_GEMM_AUTO_MODE=3
run c3F2tf c3 WINO_UFOLD=2 WINO_GEMM_AUTO_MODE=3
