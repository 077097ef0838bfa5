#!/bin/bash
# A/B of two builds on one box: libwino.so (new) vs libwino_base.so (baseline), interleaved.
# usage: bash tools/ab_lib.sh "c4,c2,c3,c5" [reps]
CFGS=${1:-c4,c2,c3,c5}; REPS=${2:-2}
mkdir -p gpurun_out
L=paper_1611_06565_b200
cp $L/libwino.so /tmp/libwino_new.so
first=${CFGS%%,*}; rest=${CFGS#*,}; [ "$rest" = "$CFGS" ] && rest=""
run() {
  timeout 300 python bench.py --config $first --extra "$rest" --steps 20 --warmup 5 --nets "" --nd "" \
    --no-cpu-baseline --no-tf32-peak > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err || { echo "$1 failed"; tail -3 gpurun_out/ab_$1.err; return; }
  python - $1 <<'PY'
import json, sys
t = sys.argv[1]
d = json.load(open("gpurun_out/ab_%s.json" % t))
for n, c in d["configs"].items():
    print("%-8s %s %.4f ms |" % (t, n, c["ms_per_layer"]), " ".join("%s=%.4f" % (s, v["ms"]) for s, v in c["stages"].items()))
PY
}
for r in $(seq $REPS); do
  cp /tmp/libwino_new.so $L/libwino.so; run new$r
  cp $L/libwino_base.so $L/libwino.so; run base$r
done
cp /tmp/libwino_new.so $L/libwino.so
