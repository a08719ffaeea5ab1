cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "bert" 2>&1 | tail -1
for lib in ab/libb2_base.so paper_2006_05096_b200/libb2.so; do
  B2_LIB=$PWD/$lib timeout 120 python tools/profile_ops.py bert 128 > gpurun_out/o.log 2>&1; echo "$lib $(head -1 gpurun_out/o.log)"; grep attention gpurun_out/o.log | head -2
  B2_LIB=$PWD/$lib timeout 120 python tools/profile_ops.py bert 1 > gpurun_out/o.log 2>&1; echo "$lib $(head -1 gpurun_out/o.log)"
done
