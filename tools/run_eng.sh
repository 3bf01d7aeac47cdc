cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | grep -E "Error|assert|passed|failed" | head -20
timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
