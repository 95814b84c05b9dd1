#!/bin/bash
# Build an experiment variant of libtrioalign_b200.so with extra nvcc flags
# into exp/<name>/ (for A/B through TA_LIB_PATH_EXPERIMENT).
# usage: tools/build_variant.sh <name> "<-DFLAG ...>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2
SRC=/tmp/ta_variant_$NAME/pkg
rm -rf "/tmp/ta_variant_$NAME"; mkdir -p "$SRC"
cp -r "$ROOT/paper_2605_28400_b200/csrc" "$ROOT/paper_2605_28400_b200/Makefile" "$SRC/"
cp -r "$ROOT/include" "/tmp/ta_variant_$NAME/include"
NV="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I$ROOT/include $FLAGS"
make -s -C "$SRC" -j"$(nproc)" NVFLAGS="$NV" ROOT="$ROOT" "$SRC/libtrioalign_b200.so" >/dev/null
mkdir -p "$ROOT/exp/$NAME"
cp "$SRC/libtrioalign_b200.so" "$ROOT/exp/$NAME/"
echo "exp/$NAME/libtrioalign_b200.so"
