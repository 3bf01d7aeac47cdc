cd $GRAFT_REPO_ROOT
TAG=_now timeout 300 python tools/engine_trace7b.py 2 2>&1 | tail -1
python tools/trace7b_report.py gpurun_out/trace7b_p2_now.npz
TAG=_now timeout 300 python tools/engine_trace7b.py 4 2>&1 | tail -1
python tools/trace7b_report.py gpurun_out/trace7b_p4_now.npz
