cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02g_tests.log
timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02g_prefill2.log 2>&1
timeout 600 python tools/prefill_profile.py > gpurun_out/r02g_prefill3.log 2>&1
timeout 300 python tools/prefill_stack.py > gpurun_out/r02g_stack.log 2>&1
