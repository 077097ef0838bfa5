#!/bin/bash
# Interleaved A/B of several builds on one box: libwino.so (default) and
# libwino_<name>.so for every name given (tools/build_variant.sh).
# usage: bash tools/ab_multi.sh "c4,c2" 2 cs cg wt
CFGS=${1:-c4}; REPS=${2:-2}; shift 2
mkdir -p gpurun_out
L=paper_1611_06565_b200
cp $L/libwino.so /tmp/libwino_default.so
first=${CFGS%%,*}; rest=${CFGS#*,}; [ "$rest" = "$CFGS" ] && rest=""
run() {
  timeout 300 python bench.py --config $first --extra "$rest" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err || { echo "$1 failed"; tail -3 gpurun_out/ab_$1.err; return; }
  python - $1 <<'PY'
import json, sys
t = sys.argv[1]
d = json.load(open("gpurun_out/ab_%s.json" % t))
for n, c in d["configs"].items():
    print("%-12s %s %.4f ms |" % (t, n, c["ms_per_layer"]), " ".join("%s=%.4f" % (s, v["ms"]) for s, v in c["stages"].items()))
PY
}
for r in $(seq $REPS); do
  cp /tmp/libwino_default.so $L/libwino.so; run default$r
  for n in "$@"; do cp $L/libwino_$n.so $L/libwino.so; run $n$r; done
done
cp /tmp/libwino_default.so $L/libwino.so
