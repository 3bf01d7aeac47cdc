cd $GRAFT_REPO_ROOT
echo "== prev code"; (cd build/wt_prev && timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error")
echo "== plain"; timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
echo "== plain again"; timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
timeout 300 python -m pytest -q -x tests/test_gpu_engine.py tests/test_gpu_tp_engine.py 2>&1 | tail -2
timeout 300 python tools/model_bench.py 2>&1 | tail -6
