# narrow-K GEMMs (MobileNet 1x1 shapes): 64-wide vs narrow A boxes
export B2_DEV=1   # developer knobs (B2_*) honoured
cd $GRAFT_REPO_ROOT
M=3211264
for s in "32 16" "16 96" "24 144" "32 192"; do python tools/gemm_micro.py $M $s; B2_NARROW_K=0 python tools/gemm_micro.py $M $s; done
