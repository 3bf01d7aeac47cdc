cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/t_model.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_configs.py -v -x --durations=0 > gpurun_out/t_configs.log 2>&1
