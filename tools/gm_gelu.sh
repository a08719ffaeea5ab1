# BERT FFN up-projection: GELU epilogue cost
export B2_DEV=1   # developer knobs (B2_*) honoured
cd $GRAFT_REPO_ROOT
for a in 0 3; do MICRO_ACT=$a python tools/gemm_micro.py 16384 768 3072; done
