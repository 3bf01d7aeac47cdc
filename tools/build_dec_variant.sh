#!/bin/bash
# variant of the DEC translation unit: build/variants/libdec_<tag>.so
set -e
TAG=$1; shift
cd /root/repo
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -warn-spills "$@" -c paper_2410_13461_b200/csrc/engine_dec.cu -o build/variants/dec_$TAG.o
OBJS=$(ls build/obj/*.o | grep -v '/engine_dec.o$')
nvcc $ARCH -shared -Xcompiler -fPIC -o build/variants/libdec_$TAG.so $OBJS build/variants/dec_$TAG.o
echo build/variants/libdec_$TAG.so
