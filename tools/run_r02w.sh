cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/gemv_one.py 4096 32000 1 2 > gpurun_out/r02w_pre.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemv -s 3 -c 1 -o gpurun_out/r02w_gemv32k_p2 python tools/gemv_one.py 4096 32000 1 2 > gpurun_out/r02w_ncu.log 2>&1
