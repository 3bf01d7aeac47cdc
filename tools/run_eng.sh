cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_tp_engine.py -q -x > gpurun_out/t_tpe.log 2>&1
export PMPD_BENCH_TP=1
PMPD_TP_ENGINE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29601 bench.py --steps 2 --warmup 3 --no-cpu --no-prefill --no-fp16 --no-model > gpurun_out/b_tpe.json 2> gpurun_out/b_tpe.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29602 bench.py --steps 2 --warmup 3 --no-cpu --no-prefill --no-fp16 --no-model > gpurun_out/b_tpn.json 2> gpurun_out/b_tpn.err
