cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
timeout 600 python -m pytest tests/test_gpu.py -q -k "batch_invariance and resnet50" 2>&1 | grep -E "assert|Error|passed|failed" | head -5
done
for cfg in "B2_DEV=1 B2_PAIR=0 B2_SPLIT=0" ""; do
 for b in 256 7 1; do
  echo "== $cfg b=$b"; env $cfg timeout 300 python tools/det_layers.py resnet50 $b 6 2>&1 | tail -3
 done
done
