#!/bin/bash
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/libeng_*.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f timeout 120 python tools/engine_trace.py 2>&1 | tail -7
  PMPD_LIB=$PWD/$f timeout 200 python tools/engine_probe.py 2>&1 | grep engine
done
