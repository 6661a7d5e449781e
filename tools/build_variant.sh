#!/bin/bash
# Build an experiment variant of libakv_sm100a.so (A/B runs select it with
# AKV_LIB=<path>): akv_decode.cu from a git revision and/or extra defines.
#   bash tools/build_variant.sh OUT.so [REV] [-DFLAG ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$1; shift
REV=""
if [ $# -gt 0 ] && [[ "$1" != -* ]]; then REV=$1; shift; fi
W=$(mktemp -d)
cp -r "$ROOT/paper_2310_01801_b200/csrc" "$W/csrc"
mkdir -p "$W/include" && cp "$ROOT/include/akv.h" "$W/include/"
if [ -n "$REV" ]; then git -C "$ROOT" show "$REV:paper_2310_01801_b200/csrc/akv_decode.cu" > "$W/csrc/akv_decode.cu"; fi
mkdir -p "$W/x/y" && mv "$W/csrc" "$W/x/y/csrc" && mv "$W/include" "$W/x/include" 2>/dev/null || true
# akv_common.cuh includes ../../include/akv.h relative to csrc
mkdir -p "$W/inc2" && cp "$ROOT/include/akv.h" "$W/x/include/akv.h"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr "$@" -c "$W/x/y/csrc/akv_decode.cu" -o "$W/akv_decode.o"
objs=""
for f in "$ROOT"/paper_2310_01801_b200/csrc/*.cu; do
  b=$(basename "$f" .cu); [ "$b" = akv_decode ] && continue; objs="$objs $ROOT/build/$b.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" $objs "$W/akv_decode.o"
rm -rf "$W"
echo "built $OUT (rev ${REV:-worktree}) $*"
