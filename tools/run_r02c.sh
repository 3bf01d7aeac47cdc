cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bounds.py tests/test_gpu_model.py -q -x > gpurun_out/r02c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02c_tests.log
timeout 600 python tools/model_bench.py 2 > gpurun_out/r02c_model2.json 2>&1
timeout 900 python tools/model_bench.py 3 > gpurun_out/r02c_model3.json 2>&1
timeout 900 bash tools/decode_sweep.sh > gpurun_out/r02c_sweep.log 2>&1
