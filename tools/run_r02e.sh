cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_model.py tests/test_gpu_configs.py tests/test_gpu_tpmodel.py -q -x > gpurun_out/r02e_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02e_tests.log
timeout 300 python tools/prefill_profile2.py 4 > gpurun_out/r02e_prefill2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_prefill2_launches.csv python tools/prefill_profile2.py 4 > gpurun_out/r02e_prefill2_ncu.log 2>&1
timeout 600 python tools/model_bench.py 2 > gpurun_out/r02e_model2.json 2>&1
