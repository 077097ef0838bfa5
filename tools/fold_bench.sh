#!/bin/bash
# A/B of the a5 epilogue fusion (WINO_FOLD=F, WINO_FOLD_RES) on the bench configs.
mkdir -p gpurun_out
run() {  # tag, env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --config c3 --extra c5,c2 --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/fold_$tag.json 2> gpurun_out/fold_$tag.err
  python - $tag <<'PY'
import json, sys
t = sys.argv[1]
d = json.load(open("gpurun_out/fold_%s.json" % t))
for n, c in d["configs"].items():
    print("%-6s %s %.4f ms  fold=%s " % (t, n, c["ms_per_layer"], c["info"].get("fold")),
          " ".join("%s=%.4f" % (s, v["ms"]) for s, v in c["stages"].items()))
PY
}
run F0 WINO_FOLD=0
run F1 WINO_FOLD=1
run F2 WINO_FOLD=2
run F1s WINO_FOLD=1 WINO_FOLD_RES=0
run F2s WINO_FOLD=2 WINO_FOLD_RES=0
