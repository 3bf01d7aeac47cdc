cd $GRAFT_REPO_ROOT
for c in 2.0 3.0 5.0; do echo "== skcost $c"; PMPD_GEMM_SKCOST=$c timeout 600 python tools/prefill_stack.py 2>&1 | tail -1 | cut -c1-120; done
