#!/bin/bash
# usage: tools/build_gemv_variant.sh <tag> [-DNAME=VAL ...] -> build/variants/libgemv_<tag>.so
set -e
TAG=$1; shift
cd "$(dirname "$0")/.."
make -s -C "$PWD/paper_2410_13461_b200/csrc" >/dev/null
mkdir -p build/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills "$@" \
  -c paper_2410_13461_b200/csrc/gemv.cu -o build/variants/gemv_$TAG.o
OBJS=$(ls build/obj/*.o | grep -v '/gemv.o$')
nvcc $ARCH -shared -Xcompiler -fPIC -o build/variants/libgemv_$TAG.so $OBJS build/variants/gemv_$TAG.o
echo build/variants/libgemv_$TAG.so
