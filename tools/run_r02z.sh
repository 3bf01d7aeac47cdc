cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemv.py tests/test_gpu_engine.py -q -x > gpurun_out/r02z_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02z_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1
