cd $GRAFT_REPO_ROOT
echo "== base"; timeout 900 python tools/model_bench.py 3 2>&1 | grep '"run": "progressive"'; timeout 600 python tools/model_bench.py 2 2>&1 | grep '"run": "progressive"'
echo "== noload"; PMPD_LIB=$PWD/build/variants/libdec_noload.so timeout 900 python tools/model_bench.py 3 2>&1 | grep '"run": "progressive"'; PMPD_LIB=$PWD/build/variants/libdec_noload.so timeout 600 python tools/model_bench.py 2 2>&1 | grep '"run": "progressive"'
