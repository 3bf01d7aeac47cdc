#!/bin/bash
# usage: tools/prof_gemv.sh <tag> <KxN> <p>   (run on the GPU box)
TAG=$1; SHAPE=$2; P=$3
python tools/gemv_probe.py --shapes $SHAPE --iters 6 --copies 2 --p $P > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:qgemv -s 5 -c 1 -o gpurun_out/prof_$TAG \
  python tools/gemv_probe.py --shapes $SHAPE --iters 6 --copies 2 --p $P > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
