cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu.py -q -x -k "fullsize or batch_invariance" 2>&1 | grep -E "^E |assert|passed|failed" | head -12
done
bash tools/r3_ncu_bert.sh
