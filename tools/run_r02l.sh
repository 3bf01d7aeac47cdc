cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02l_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02l_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02l_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err
timeout 900 python tools/model_bench.py 3 > gpurun_out/r02l_model3.json 2>&1
