# narrow-N memory-bound GEMM (MobileNet 112x112x32 -> 16): which epilogue step paces the tiles
cd $GRAFT_REPO_ROOT
M=3211264
for e in 0 1 3 4 5 6; do B2_EPI_MODE=$e python tools/gemm_micro.py $M 32 16; done
for e in 0 1 4 5; do B2_EPI_MODE=$e python tools/gemm_micro.py 802816 64 64; done
