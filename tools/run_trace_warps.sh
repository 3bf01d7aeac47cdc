#!/bin/bash
cd $GRAFT_REPO_ROOT
for f in build/variants/libeng_*.so; do
  tag=$(basename $f .so)
  echo "== $tag"
  PMPD_LIB=$PWD/$f TAG=_$tag timeout 300 python tools/engine_trace7b.py 2 2>&1 | tail -1
  python tools/trace_warps_report.py gpurun_out/trace7b_p2_$tag.npz
  PMPD_LIB=$PWD/$f TAG=_$tag timeout 300 python tools/engine_trace7b.py 4 2>&1 | tail -1
  python tools/trace_warps_report.py gpurun_out/trace7b_p4_$tag.npz
done
