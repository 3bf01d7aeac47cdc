cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/r02t_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02t_tests.log
