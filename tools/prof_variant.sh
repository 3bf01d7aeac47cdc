#!/bin/bash
# usage: tools/prof_variant.sh <tag> <lib> <KxN> <p>
TAG=$1; LIB=$2; SHAPE=$3; P=$4
PMPD_LIB=$PWD/$LIB python tools/gemv_probe.py --shapes $SHAPE --iters 6 --copies 2 --p $P > /dev/null 2>&1 && \
PMPD_LIB=$PWD/$LIB ncu --set full --clock-control none --import-source on -k regex:qgemv -s 5 -c 1 -o gpurun_out/prof_$TAG \
  python tools/gemv_probe.py --shapes $SHAPE --iters 6 --copies 2 --p $P > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
