#!/bin/bash
# Prefill GEMM tile-configuration sweep (PMPD_GEMM_CFG="ng,mb", PMPD_GEMM_SPLITK=S) on the config-4 shapes
# (f32 outputs, as the model runner uses them).
cd "$(dirname "$0")/.."
for c in default 1,1 1,2 1,4 2,1 2,2 2,4 4,1 4,2; do
  for sk in 1 2 4; do
    echo "== cfg $c sk $sk"
    if [ $c = default ]; then [ $sk = 1 ] && timeout 300 python tools/gemm_bench.py 2>&1 | grep -v cublas | grep "\"p\": 4";
    else PMPD_GEMM_CFG=$c PMPD_GEMM_SPLITK=$sk timeout 300 python tools/gemm_bench.py 2>&1 | grep -v cublas | grep "\"p\": 4"; fi
  done
done
