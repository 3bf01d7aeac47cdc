cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | grep -E "Error|assert|passed|failed" | head -20
for p in 2 4; do timeout 300 python tools/engine_trace7b.py $p; done
python tools/trace7b_report.py
