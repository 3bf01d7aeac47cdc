cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/r02u_torchrun1.json 2> gpurun_out/r02u_torchrun1.err
echo "rc=$?" >> gpurun_out/r02u_torchrun1.err
