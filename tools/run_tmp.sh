cd $GRAFT_REPO_ROOT
bash tools/run_var.sh
PMPD_LIB=$PWD/build/variants/libeng_prod2.so timeout 600 python -m pytest -q -x tests/test_gpu_engine.py 2>&1 | tail -2
