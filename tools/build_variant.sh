#!/bin/bash
# Build libjz.so with one source file compiled with extra flags: tools/build_variant.sh <file.cu> <out.so> [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
src=$1; out=$2; shift 2
b=$(basename "$src" .cu)
tmp=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Iinclude "$@" -c "$src" -o $tmp/$b.o
objs=""
for f in paper_2510_27002_b200/lib/obj/*.o; do [ "$(basename $f)" = "$b.o" ] || objs="$objs $f"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$out" $tmp/$b.o $objs -Xcompiler -fPIC -lpthread -ldl -lrt
rm -rf $tmp
