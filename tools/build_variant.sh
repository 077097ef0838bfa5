#!/bin/bash
# Build a variant library for an interleaved A/B on one box (tools/ab_multi.sh):
# recompiles the listed translation units with extra -D flags into a separate
# object directory and links them with the default objects of the rest.
# usage: bash tools/build_variant.sh NAME "-DWINO_VPUT_MODE=1" xform_in_const.cu [more.cu ...]
set -e
NAME=$1; DEFS=$2; shift 2
L=paper_1611_06565_b200; O=$L/_obj_$NAME; mkdir -p $O
python -c "from paper_1611_06565_b200 import _build; _build.build()" > /dev/null
OBJS=""
for f in $L/_obj/*.o; do OBJS="$OBJS $f"; done
for src in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I $L/csrc -I include $DEFS -c $L/csrc/$src -o $O/$src.o &
  OBJS=${OBJS/$L\/_obj\/$src.o/$O\/$src.o}
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/libwino_$NAME.so $OBJS -cudart static
echo built $L/libwino_$NAME.so
