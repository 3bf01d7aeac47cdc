cd $GRAFT_REPO_ROOT
for i in 1 2; do
echo "== base"; timeout 600 python tools/model_bench.py 2 2>&1 | grep '"run": "progressive"'
echo "== pre"; PMPD_LIB=$PWD/build/variants/libdec_pre.so timeout 600 python tools/model_bench.py 2 2>&1 | grep '"run": "progressive"'
done
PMPD_LIB=$PWD/build/variants/libdec_pre.so timeout 900 python tools/model_bench.py 3 2>&1 | grep '"run": "progressive"'
PMPD_LIB=$PWD/build/variants/libdec_pre.so timeout 600 python -m pytest -q -x tests/test_gpu_model.py tests/test_gpu_configs.py 2>&1 | tail -2
