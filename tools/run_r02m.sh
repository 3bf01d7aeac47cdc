cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for s in "512 4096 12288" "512 4096 4096" "512 4096 22016" "512 11008 4096" "512 4096 32000" "128 2048 6144" "128 2048 2048" "128 2048 11264" "128 5632 2048" "128 2048 32000"; do
  timeout 300 python tools/gemm_probe.py $s
done > gpurun_out/r02m_probe.log 2>&1
