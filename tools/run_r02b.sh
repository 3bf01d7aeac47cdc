cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02b_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout 1500 bash tools/sanitize.sh
