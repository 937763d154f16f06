#!/bin/bash
# Build an A/B variant of libstable_b200.so with extra nvcc flags for ONE source file:
#   tools/build_variant.sh NAME SRC "FLAGS"   ->  alt_libs/NAME.so (git-ignored; load it with
#   STABLE_B200_LIB=alt_libs/NAME.so).  The other objects come from the main build.
set -e
name=$1; src=$2; flags=$3
here=$(cd "$(dirname "$0")/.." && pwd)
pkg=$here/paper_2604_01617_b200
make -s -C "$pkg" >/dev/null
tmp=$(mktemp -d)
cp "$pkg"/build/*.o "$tmp"/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v -prec-div=true -prec-sqrt=true $flags -c "$pkg/csrc/$src.cu" -o "$tmp/$src.o" 2> "$tmp/$src.ptxas.log" \
  || (cat "$tmp/$src.ptxas.log"; exit 1)
mkdir -p "$here/alt_libs"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$here/alt_libs/$name.so" "$tmp"/*.o \
  -lcudart_static -lrt -lpthread -ldl
grep -A2 "route_kernelILi4ELb0" "$tmp/$src.ptxas.log" | grep -E "registers|spill" || true
rm -rf "$tmp"
