cd $GRAFT_REPO_ROOT
timeout 900 python tools/calib_probe.py
