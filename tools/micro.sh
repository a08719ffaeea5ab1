cd $GRAFT_REPO_ROOT
for st in 2 4 8; do B2_STAGES=$st timeout 60 python tools/conv_micro.py 256 56 56 64 64 3 1; done
B2_EPI_MODE=1 timeout 60 python tools/conv_micro.py 256 56 56 64 64 3 1
for st in 4 8; do B2_STAGES=$st timeout 60 python tools/conv_micro.py 256 224 224 8 64 7 2; done
timeout 60 python tools/conv_micro.py 256 14 14 256 256 3 1
