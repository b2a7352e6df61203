#!/bin/bash
# Build a diagnostic / experimental variant of libtccd.so into exp/:
#   tools/build_variant.sh <name> [-DMACRO=...]...   ->  exp/lib_<name>.so
# (select it with TCCD_LIB=exp/lib_<name>.so; the product build is `make`)
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
name="$1"; shift
cd "$ROOT/paper_2009_13349_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I"$ROOT/include" --fmad=false "$@" -shared -o "$ROOT/exp/lib_${name}.so" tccd.cu broad.cu irf.cu mirror.cu
