# small-K / small-N GEMM diagnosis (MobileNetV2 1x1 shapes, M = 256*112*112)
export B2_DEV=1   # developer knobs (B2_*) honoured
cd $GRAFT_REPO_ROOT
M=3211264
for s in "16 96" "24 144" "32 192" "32 16" "64 256" "64 64"; do python tools/gemm_micro.py $M $s; B2_EPI_BUFS=2 python tools/gemm_micro.py $M $s; done
