cd $GRAFT_REPO_ROOT
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_pf0.so build/variants/libeng_pf1.so build/variants/libeng_pf3.so build/variants/libeng_pf4.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
done
PMPD_LIB= timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_gemm.py tests/test_gpu_tpmodel.py -q -x 2>&1 | tail -3
