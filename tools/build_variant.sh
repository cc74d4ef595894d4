#!/bin/bash
# Build a tuning variant of libxsp.so with extra -D flags on one source file:
#   tools/build_variant.sh NAME SRC "-DXSP_FOO=0 ..."   ->  paper_1908_06869_b200/lib/libxsp_NAME.so
# (A/B on one box: XSP_LIB=$PWD/paper_1908_06869_b200/lib/libxsp_NAME.so python bench.py ...)
set -e
NAME=$1; SRC=$2; DEFS=$3
D=$(cd "$(dirname "$0")/../paper_1908_06869_b200" && pwd)
make -C "$D" -s
OBJ=$D/lib/obj
FMAD=""
case $SRC in analyze|leveled) FMAD="-fmad=false";; esac
nvcc -std=c++20 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  -I"$D/../include" -I"$D/csrc" $FMAD $DEFS -c "$D/csrc/$SRC.cu" -o "$OBJ/${SRC}_$NAME.o"
OBJS=""
for o in correlate analyze leveled sort validate resolve capi pipeline report combine ingest packed; do
  if [ "$o" = "$SRC" ]; then OBJS="$OBJS $OBJ/${SRC}_$NAME.o"; else OBJS="$OBJS $OBJ/$o.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$D/lib/libxsp_$NAME.so" $OBJS -lcudart -ldl
echo "$D/lib/libxsp_$NAME.so"
