#!/bin/bash
B=./tools/microbench/stream_bench
$B
for g in 1 2; do for sb in 4096 8192 16384 32768; do for ns in 2 4 8 16; do
  tot=$((sb*ns)); if [ $g = 1 ] && [ $tot -gt 200000 ]; then continue; fi; if [ $g = 2 ] && [ $tot -gt 100000 ]; then continue; fi
  timeout 20 $B $g $sb $ns 1 || echo "FAILED $g $sb $ns"
done; done; done
