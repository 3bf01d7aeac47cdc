#!/bin/bash
# Times every build/variants/libeng_*.so (plus the default library) with engine_probe and checks parity
# with the engine tests.  usage: tools/engine_variants.sh
cd "$(dirname "$0")/.."
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_*.so; do
  tag=$(basename $f .so)
  echo "== $tag"
  PMPD_LIB=$PWD/$f timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1
  PMPD_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
done
