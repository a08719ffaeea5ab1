# narrow-N memory-bound GEMM (MobileNet 112x112x32 -> 16): what paces the tiles
cd $GRAFT_REPO_ROOT
M=3211264
python tools/gemm_micro.py $M 32 16
B2_EPI_MODE=1 python tools/gemm_micro.py $M 32 16
B2_STAGES=4 python tools/gemm_micro.py $M 32 16
B2_STAGES=2 python tools/gemm_micro.py $M 32 16
B2_PDL=0 python tools/gemm_micro.py $M 32 16
