#!/bin/bash
# engine_probe + engine trace for the default library and every build/variants/libeng_*.so
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_*.so; do
  tag=$(basename $f .so)
  echo "== $tag"
  PMPD_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error|error"
  PMPD_LIB=$PWD/$f timeout 120 python tools/engine_trace.py 2 > /dev/null 2>&1 && cp gpurun_out/engine_trace.npz gpurun_out/trace_$tag.npz
done
