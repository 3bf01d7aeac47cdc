cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02r_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02r_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02r_ref.json 2> gpurun_out/r02r_ref.err
