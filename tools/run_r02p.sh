cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000
for rep in 1 2; do for m in 1 2 4 8; do
  timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,2 --shapes $S | sed 's/^/NEW /'
  PMPD_LIB=build/variants/libgemv_rowwise.so timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,2 --shapes $S | sed 's/^/OLD /'
done; done > gpurun_out/r02p_ab.log 2>&1
