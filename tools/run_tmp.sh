cd $GRAFT_REPO_ROOT
timeout 600 python tools/decoder_trace.py 2 2 2>&1 | tail -7
timeout 600 python tools/model_bench.py 2>&1 | grep '"run"'
timeout 900 python -m pytest -q -x tests/test_gpu_model.py tests/test_gpu_configs.py 2>&1 | tail -2
