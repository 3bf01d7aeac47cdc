cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_bounds.py -q -x > gpurun_out/r02s_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02s_tests.log
S=4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000
for rep in 1 2; do for m in 8; do
  timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,2 --shapes $S | sed 's/^/NEW /'
  PMPD_LIB=build/variants/libgemv_noxs2.so timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,2 --shapes $S | sed 's/^/OLD /'
done; done > gpurun_out/r02s_ab.log 2>&1
