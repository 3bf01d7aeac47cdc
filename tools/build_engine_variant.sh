#!/bin/bash
# usage: tools/build_engine_variant.sh <tag> [-DNAME=VAL ...]
# Builds build/variants/libeng_<tag>.so = the library with engine.cu recompiled under extra -D flags.
set -e
TAG=$1; shift
cd "$(dirname "$0")/.."
make -s -C "$PWD/paper_2410_13461_b200/csrc" >/dev/null
mkdir -p build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_2410_13461_b200/csrc/engine.cu -o build/variants/eng_$TAG.o
OBJS=$(ls build/obj/*.o | grep -v '/engine.o$')
nvcc $ARCH -shared -Xcompiler -fPIC -o build/variants/libeng_$TAG.so $OBJS build/variants/eng_$TAG.o
echo build/variants/libeng_$TAG.so
