cd $GRAFT_REPO_ROOT
timeout 900 python tools/gemm_bench.py > gpurun_out/gb_r2.log 2>&1
PMPD_GEMM_SERIAL_REDUCE=1 timeout 900 python tools/gemm_bench.py > gpurun_out/gb_r2s.log 2>&1
