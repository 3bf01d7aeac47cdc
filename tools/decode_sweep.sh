#!/bin/bash
# BASELINE config-4 decode sweep: pmpd_gemv per shape (K x N), batch m = 1/2/4/8, p = 4/3/2, CUDA graph of
# rotating weight copies (> 400 MB per replay, so every launch streams from HBM).
cd "$(dirname "$0")/.."
for m in 1 2 4 8; do
  timeout 600 python tools/gemv_probe.py --graph --m $m --p 4,3,2 \
    --shapes 4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000
done
