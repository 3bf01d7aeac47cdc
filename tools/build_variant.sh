#!/bin/bash
# usage: tools/build_variant.sh <source.cu basename> <tag> [-DNAME=VAL ...]
# Builds build/variants/lib<src>_<tag>.so = the library with that one source recompiled under extra -D flags.
set -e
SRC=$1; TAG=$2; shift 2
cd "$(dirname "$0")/.."
make -s -C "$PWD/paper_2410_13461_b200/csrc" >/dev/null
mkdir -p build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_2410_13461_b200/csrc/$SRC.cu -o build/variants/${SRC}_$TAG.o
OBJS=$(ls build/obj/*.o | grep -v "/$SRC.o\$")
nvcc $ARCH -shared -Xcompiler -fPIC -o build/variants/lib${SRC}_$TAG.so $OBJS build/variants/${SRC}_$TAG.o
echo build/variants/lib${SRC}_$TAG.so
