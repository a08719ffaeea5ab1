cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "mobilenet" 2>&1 | tail -1
timeout 120 python tools/profile_ops.py mobilenet_v2 256 > gpurun_out/ops_mb.log 2>&1; head -1 gpurun_out/ops_mb.log
