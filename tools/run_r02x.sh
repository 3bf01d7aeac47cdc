cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000
for rep in 1 2; do
  timeout 300 python tools/gemv_probe.py --graph --m 1 --p 4,2 --shapes $S | sed 's/^/BASE /'
  for v in ncw12 tpw3 ncw16; do
    PMPD_LIB=build/variants/libgemv_$v.so timeout 300 python tools/gemv_probe.py --graph --m 1 --p 4,2 --shapes $S | sed "s/^/$v /"
  done
done > gpurun_out/r02x_ab.log 2>&1
