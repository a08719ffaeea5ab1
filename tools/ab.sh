cd $GRAFT_REPO_ROOT
export B2_DEV=1   # developer knobs (B2_*) honoured
timeout 600 python tools/dbg_layerwise.py resnet50 0 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "parity" 2>&1 | tail -2
MICRO_DTYPE=0 timeout 120 python tools/gemm_micro.py 16384 4096 4096
timeout 300 python tools/profile_ops.py resnet50 64 0 | head -1
