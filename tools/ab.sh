cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "bert or toy" 2>&1 | tail -1
for fk in 512 1024; do
  B2_FOLD_MAX_K=$fk timeout 120 python tools/profile_ops.py bert 128 > gpurun_out/ops_b$fk.log 2>&1; head -1 gpurun_out/ops_b$fk.log; sed -n 2,12p gpurun_out/ops_b$fk.log
done
