#!/bin/bash
# instruction count + duration of one kernel (regex $1) of config $2 for libwino.so vs libwino_base.so
K=${1:-k_input}; C=${2:-c4}
L=paper_1611_06565_b200
cp $L/libwino.so /tmp/libwino_new.so
for v in new base; do
  [ $v = base ] && cp $L/libwino_base.so $L/libwino.so
  timeout 300 ncu --clock-control none -k regex:$K -s 3 -c 1 --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed \
    python bench.py --steps 2 --warmup 3 --config $C --extra "" --nets "" --nd "" --no-cpu-baseline --no-tf32-peak 2>/dev/null | grep -E 'inst_executed|duration|issue_active' | sed "s/^/$v /"
done
cp /tmp/libwino_new.so $L/libwino.so
