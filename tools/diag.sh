#!/bin/bash
# One-call diagnostic sweep on the GPU box: microbenchmarks + engine variants + per-op timeline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
echo "=== tile_bench"; timeout 60 ./tools/microbench/tile_bench
echo "=== mma_tput"; timeout 60 ./tools/microbench/mma_tput
echo "=== stream_bench"; timeout 60 ./tools/microbench/stream_bench 1 24576 8 3; timeout 60 ./tools/microbench/stream_bench 1 16384 12 3
} > gpurun_out/diag_micro.log 2>&1
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_*.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error|error"
done > gpurun_out/diag_variants.log 2>&1
timeout 300 python tools/engine_trace.py > gpurun_out/diag_trace.log 2>&1
echo diag done
