#!/bin/bash
for f in paper_2410_13461_b200/lib/libpmpd_b200.so build/variants/lib_*.so; do
  echo "== $f"
  PMPD_LIB=$PWD/$f python tools/gemv_probe.py --graph --shapes 4096x4096,4096x22016,4096x32000 --p 2,4 2>&1 | grep -v copies=0
done
