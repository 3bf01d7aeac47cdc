cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_bounds.py tests/test_gpu_tp.py tests/test_gpu_model.py -q -x > gpurun_out/r02o_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02o_tests.log
timeout 900 bash tools/decode_sweep.sh > gpurun_out/r02o_sweep.log 2>&1
