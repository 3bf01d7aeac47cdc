cd $GRAFT_REPO_ROOT
timeout 600 python tools/decoder_trace.py 2 2 2>&1 | tail -7
timeout 600 python tools/decoder_trace.py 3 2 2>&1 | tail -7
