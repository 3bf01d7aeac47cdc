cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_search.py tests/test_gpu_model.py tests/test_gpu_tpmodel.py -q > gpurun_out/t_new.log 2>&1
timeout 300 python tools/prefill_stack.py > gpurun_out/prefill.log 2>&1
