#!/bin/bash
# Prefill GEMM tile-configuration sweep (PMPD_GEMM_CFG="ng,mb") on the config-4 shapes.
cd "$(dirname "$0")/.."
for c in default 1,1 1,2 1,4 2,1 2,2 2,4 4,1 4,2; do
  echo "== cfg $c"
  if [ $c = default ]; then timeout 300 python tools/gemm_bench.py 2>&1 | grep -v cublas | grep "\"p\": 4";
  else PMPD_GEMM_CFG=$c timeout 300 python tools/gemm_bench.py 2>&1 | grep -v cublas | grep "\"p\": 4"; fi
done
