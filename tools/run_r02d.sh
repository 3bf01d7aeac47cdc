cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_bounds.py tests/test_gpu_tp.py -q -x > gpurun_out/r02d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02d_tests.log
for m in 1 4; do timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,3,2 --shapes 4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000; done > gpurun_out/r02d_sweep.log 2>&1
timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02d_prefill2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_prefill2_launches.csv python tools/prefill_profile2.py 4 > gpurun_out/r02d_prefill2_ncu.log 2>&1
