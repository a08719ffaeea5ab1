cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -k "band8 or conv3x3" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "vgg" 2>&1 | tail -1
timeout 60 python tools/conv_micro.py 256 224 224 3 64 3 1
timeout 120 python tools/profile_ops.py vgg16 256 2>/dev/null | head -4
