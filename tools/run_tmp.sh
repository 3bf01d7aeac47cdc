cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err; tail -2 gpurun_out/b_e2e.err
