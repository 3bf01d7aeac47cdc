cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/r02j_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02j_tests.log
timeout 300 python tools/prefill_stack.py > gpurun_out/r02j_stack.log 2>&1
PMPD_GEMM_DSM=0 timeout 300 python tools/prefill_stack.py > gpurun_out/r02j_stack_nodsm.log 2>&1
PMPD_GEMM_SKCOST=0.5 timeout 300 python tools/prefill_stack.py > gpurun_out/r02j_stack_sk0.5.log 2>&1
timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02j_prefill2.log 2>&1
PMPD_GEMM_DSM=0 timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02j_prefill2_nodsm.log 2>&1
timeout 600 python tools/gemm_bench.py > gpurun_out/r02j_gemm_bench.log 2>&1
PMPD_GEMM_DSM=0 timeout 600 python tools/gemm_bench.py > gpurun_out/r02j_gemm_bench_nodsm.log 2>&1
