cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bounds.py tests/test_gpu_model.py -q -x > gpurun_out/r02f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02f_tests.log
timeout 300 python tools/prefill_stack.py > gpurun_out/r02f_stack.log 2>&1
PMPD_GEMM_PDL_OFF=1 true
timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02f_prefill2.log 2>&1
timeout 600 python tools/prefill_profile.py > gpurun_out/r02f_prefill3.log 2>&1
timeout 600 python tools/gemm_bench.py > gpurun_out/r02f_gemm_bench.log 2>&1
