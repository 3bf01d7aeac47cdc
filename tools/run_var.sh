cd $GRAFT_REPO_ROOT
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_*.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
done
