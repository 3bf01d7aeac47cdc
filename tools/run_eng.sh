cd $GRAFT_REPO_ROOT
timeout 900 python tools/model_bench.py 2 > gpurun_out/mb2.log 2>&1
timeout 1500 python tools/model_bench.py 3 > gpurun_out/mb3.log 2>&1
