cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_tp_engine.py tests/test_gpu_engine.py tests/test_gpu_loader.py tests/test_gpu_model.py -q -x > gpurun_out/t_tpe.log 2>&1
timeout 300 python tools/engine_probe.py > gpurun_out/probe.log 2>&1
