cd $GRAFT_REPO_ROOT
for fl in 1 0 2 3; do
  echo "== flush $fl"
  PMPD_ENGINE_PART_FLUSH=$fl timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
done
echo "== even"
PMPD_ENGINE_EVEN=1 timeout 300 python tools/engine_probe.py 2>&1 | grep -E "engine|Error"
