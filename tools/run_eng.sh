cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_model.py tests/test_gpu_glue.py -q -x > gpurun_out/t_model.log 2>&1
timeout 300 python tools/decoder_trace.py 3 2 > gpurun_out/dtrace.log 2>&1
timeout 300 python tools/decoder_trace.py 2 2 >> gpurun_out/dtrace.log 2>&1
