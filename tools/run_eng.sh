cd $GRAFT_REPO_ROOT
for p in 2 4; do timeout 300 python tools/engine_trace7b.py $p; done
python tools/trace7b_report.py
