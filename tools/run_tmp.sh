cd $GRAFT_REPO_ROOT
bash tools/run_var.sh
bash tools/run_var.sh
timeout 300 python tools/model_bench.py 2 2>&1 | grep '"run": "progressive"'
timeout 600 python -m pytest -q -x tests/test_gpu_engine.py tests/test_gpu_model.py 2>&1 | tail -2
