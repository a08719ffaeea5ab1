# ResNet expand 1x1 (+residual): narrow (N=64 slice) fold vs full-width identity fold
export B2_DEV=1   # developer knobs (B2_*) honoured
cd $GRAFT_REPO_ROOT
for s in "50176 256 1024" "200704 128 512" "12544 512 2048" "802816 64 256"; do
python tools/gemm_micro.py $s res; B2_FOLD_N64=0 python tools/gemm_micro.py $s res; done
