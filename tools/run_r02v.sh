cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PMPD_BENCH_TP=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/r02v_tp1.json 2> gpurun_out/r02v_tp1.err
echo "rc=$?" >> gpurun_out/r02v_tp1.err
PMPD_BENCH_TP=1 PMPD_TP_ENGINE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/r02v_tp1_perop.json 2> gpurun_out/r02v_tp1_perop.err
echo "rc=$?" >> gpurun_out/r02v_tp1_perop.err
