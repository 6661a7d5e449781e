#!/bin/bash
# Build an experiment variant of libakv_sm100a.so (A/B runs select it with
# AKV_LIB=<path>): any csrc file taken from a git revision, extra defines.
#   bash tools/build_variant.sh OUT.so [akv_decode.cu@REV ...] [-DFLAG ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$1; shift
W=$(mktemp -d)
mkdir -p "$W/pkg/csrc" "$W/include"
cp "$ROOT"/paper_2310_01801_b200/csrc/* "$W/pkg/csrc/"
cp "$ROOT/include/akv.h" "$W/include/"
while [ $# -gt 0 ] && [[ "$1" == *@* ]]; do
  f=${1%@*}; rev=${1#*@}
  git -C "$ROOT" show "$rev:paper_2310_01801_b200/csrc/$f" > "$W/pkg/csrc/$f"
  shift
done
objs=""
for f in "$W"/pkg/csrc/*.cu; do
  b=$(basename "$f" .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c "$f" -o "$W/$b.o" &
  objs="$objs $W/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" $objs
rm -rf "$W"
echo "built $OUT"
