#!/bin/bash
# engine_probe + 7B token trace (p=2) for the default library and every build/variants/libeng_*.so
cd $GRAFT_REPO_ROOT
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_*.so; do
  tag=$(basename $f .so)
  echo "== $tag"
  PMPD_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
  PMPD_LIB=$PWD/$f TAG=_$tag timeout 300 python tools/engine_trace7b.py 2 2>&1 | tail -1
  python tools/trace7b_report.py gpurun_out/trace7b_p2_$tag.npz
done
