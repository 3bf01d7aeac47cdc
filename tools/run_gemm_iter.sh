#!/bin/bash
# GPU job for one prefill-GEMM iteration: parity tests, config probe, 7B stack, optional ncu (NCU=1)
cd "$(dirname "$0")/.."
O=gpurun_out/gemm_iter; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
timeout 300 python tools/gemm_probe.py 512 4096 4096 default 4,2,4 2,2,2 4,1,2 2,1,1 4,2,1
timeout 300 python tools/gemm_probe.py 2048 4096 4096 default 2,4,1
timeout 300 python tools/prefill_stack.py 2>&1 | tail -1
if [ "$NCU" = 1 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o $O/gemm2048 python tools/gemm_one.py 2048 4096 4096 > $O/ncu2048.log 2>&1
  ncu -i $O/gemm2048.ncu-rep --page source --csv --print-source sass > $O/sass2048.csv 2>/dev/null
fi
