cd $GRAFT_REPO_ROOT
export B2_DEV=1   # developer knobs (B2_*) honoured
for st in 2 4 8; do B2_STAGES=$st timeout 60 python tools/conv_micro.py 256 56 56 64 64 3 1; done
timeout 60 python tools/gemm_micro.py 802816 576 64
timeout 60 python tools/gemm_micro.py 802816 576 128
timeout 60 python tools/conv_micro.py 256 56 56 64 128 3 1
timeout 60 python tools/conv_micro.py 256 28 28 128 128 3 1
B2_EPI_MODE=1 timeout 60 python tools/conv_micro.py 256 56 56 64 64 3 1
