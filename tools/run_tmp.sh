cd $GRAFT_REPO_ROOT
for v in lo lodbl; do
PMPD_LIB=$PWD/build/variants/libeng_$v.so TAG=_$v timeout 300 python tools/engine_trace7b.py 2 2>&1 | tail -1
python tools/trace7b_report.py gpurun_out/trace7b_p2_$v.npz | tail -4
done
