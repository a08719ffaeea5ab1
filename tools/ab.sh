cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -k "pointwise" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "mobilenet" 2>&1 | tail -1
for pw in 0 1; do B2_PWS=$pw timeout 120 python tools/profile_ops.py mobilenet_v2 256 > gpurun_out/mb$pw.log 2>&1; head -1 gpurun_out/mb$pw.log; done
