cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bounds.py -q -x > gpurun_out/r02i_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02i_tests.log
timeout 300 python tools/prefill_stack.py > gpurun_out/r02i_stack.log 2>&1
PMPD_GEMM_DSM=0 timeout 300 python tools/prefill_stack.py > gpurun_out/r02i_stack_nodsm.log 2>&1
for c in 0.2 0.5 1.0; do PMPD_GEMM_SKCOST=$c timeout 300 python tools/prefill_stack.py > gpurun_out/r02i_stack_sk$c.log 2>&1; done
timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02i_prefill2.log 2>&1
PMPD_GEMM_SKCOST=0.3 timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02i_prefill2_sk.log 2>&1
timeout 600 python tools/gemm_bench.py > gpurun_out/r02i_gemm_bench.log 2>&1
