cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/gemv_one.py 4096 11008 1 4 > gpurun_out/r02k_pre.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemv -s 3 -c 1 -o gpurun_out/r02k_gemv_p4 python tools/gemv_one.py 4096 11008 1 4 > gpurun_out/r02k_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qgemv -s 3 -c 1 -o gpurun_out/r02k_gemv_p2 python tools/gemv_one.py 4096 11008 1 2 > gpurun_out/r02k_ncu2.log 2>&1
