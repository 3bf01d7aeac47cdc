cd $GRAFT_REPO_ROOT
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_db.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f timeout 300 python tools/decoder_trace.py 3 2 2>&1 | grep -v -i "warn\|nanmax"
  PMPD_LIB=$PWD/$f timeout 300 python tools/decoder_trace.py 2 2 2>&1 | grep -v -i "warn\|nanmax" | head -4
done
