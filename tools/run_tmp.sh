cd $GRAFT_REPO_ROOT
PMPD_BENCH_TP=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > gpurun_out/b_tp1.json 2> gpurun_out/b_tp1.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-prefill > gpurun_out/b_1.json 2> gpurun_out/b_1.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
