cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x > gpurun_out/t_engine.log 2>&1
timeout 400 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/t_model.log 2>&1
timeout 300 python tools/engine_probe.py > gpurun_out/probe.log 2>&1
