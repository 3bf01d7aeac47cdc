cd $GRAFT_REPO_ROOT
echo "== prev code"; (cd build/wt_prev && timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error")
echo "== plain"; timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
echo "== paired"; PMPD_ENGINE_PAIRED=1 timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
timeout 300 python -m pytest -q -x tests/test_gpu_engine.py 2>&1 | tail -2
