cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in 1 2 4 8; do
  timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,2 --shapes 4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000,2048x2048,2048x6144,2048x11264
  PMPD_GEMV_SPLITK=1 timeout 300 python tools/gemv_probe.py --graph --m $m --p 4,2 --shapes 4096x4096,4096x11008,11008x4096,5632x2048,2048x5632,4096x32000,2048x2048,2048x6144,2048x11264 | sed 's/^/SPLITK /'
done > gpurun_out/r02n_grid.log 2>&1
