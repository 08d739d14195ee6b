#!/bin/bash
# Builds variants/libgdx_<name>.so: the current objects of libgdx with
# one translation unit recompiled with extra flags (e.g. a -D knob), for
# same-box A/B runs with tools/ab_libs.sh.
#   tools/build_variant.sh <name> <unit: sssp|pagerank|tc|bc|...> [nvcc flags...]
# SRC=<file.cu> compiles that file (e.g. the unit at an older commit, copied
# next to the sources) in place of <unit>.cu.
set -eu
name=$1; unit=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_2401_02472_b200/csrc
OBJ=$ROOT/build/gdx
OUT=$ROOT/variants
make -C "$CSRC" -j8 > /dev/null
mkdir -p "$OUT"
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c "${SRC:-$CSRC/$unit.cu}" -o "$OUT/$unit.$name.o"
objs=""
for u in api build sssp pagerank tc bc edgelist refstream multi textbook; do
    if [ "$u" = "$unit" ]; then objs="$objs $OUT/$unit.$name.o"; else objs="$objs $OBJ/$u.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libgdx_$name.so" \
    $objs -Xlinker -z,defs -lpthread -ldl -lrt
rm "$OUT/$unit.$name.o"
echo "$OUT/libgdx_$name.so"
