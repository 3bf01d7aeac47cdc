cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/gemm_one.py 512 4096 4096 > gpurun_out/r02h_pre.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r02h_gemm512 python tools/gemm_one.py 512 4096 4096 > gpurun_out/r02h_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r02h_gemm128 python tools/gemm_one.py 128 2048 2048 > gpurun_out/r02h_ncu2.log 2>&1
