cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -q -x tests/test_gpu_model.py tests/test_gpu_configs.py tests/test_gpu_engine.py tests/test_gpu_glue.py 2>&1 | tail -2
for i in 1 2; do timeout 600 python tools/model_bench.py 2 2>&1 | grep '"run"'; done
timeout 900 python tools/model_bench.py 3 2>&1 | grep '"run"'
