cd $GRAFT_REPO_ROOT
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_evn.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f timeout 300 python tools/l2_probe.py 2>&1 | grep -E "L=|Error"
done
