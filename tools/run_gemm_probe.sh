#!/bin/bash
# GPU job: prefill GEMM configuration probe + variants + ncu of the default launch
cd "$(dirname "$0")/.."
O=gpurun_out/gemm_probe; mkdir -p $O
timeout 300 python tools/gemm_probe.py 512 4096 4096 > $O/m512_4096.jsonl 2>&1
timeout 300 python tools/gemm_probe.py 2048 4096 4096 default 4,2,1 2,4,1 4,1,1 2,2,1 > $O/m2048_4096.jsonl 2>&1
timeout 300 python tools/gemm_probe.py 512 4096 11008 default 4,2,1 4,2,2 2,4,2 4,1,2 2,2,2 > $O/m512_4096x11008.jsonl 2>&1
for v in nodq nomma nb2; do
  PMPD_LIB=build/variants/libgemm_$v.so timeout 300 python tools/gemm_probe.py 512 4096 4096 default 4,2,1 4,2,4 2,2,4 1,1,1 4,1,1 > $O/v_$v.jsonl 2>&1
  PMPD_LIB=build/variants/libgemm_$v.so timeout 300 python tools/gemm_probe.py 2048 4096 4096 default 4,2,1 > $O/v2048_$v.jsonl 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm512 python tools/gemm_one.py 512 4096 4096 > $O/ncu512.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm2048 python tools/gemm_one.py 2048 4096 4096 > $O/ncu2048.log 2>&1
ls -la $O
