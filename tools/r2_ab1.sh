# A/B matrix of kernel-selection knobs on ResNet-50 b=256 (graph-replayed forward)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { AB_LABEL="$1" env B2_DEV=1 $2 timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab1.log 2>&1; }
run default ""
run fold128 "B2_FOLD_MAX_K=128"
run fold0 "B2_FOLD_MAX_K=0"
run fold256 "B2_FOLD_MAX_K=256"
run nochain "B2_CHAIN=0"
run nopair "B2_PAIR=0"
run nodsfold "B2_DS_FOLD=0"
run fold128_nodsfold "B2_FOLD_MAX_K=128 B2_DS_FOLD=0"
B2_DEV=1 B2_FOLD_MAX_K=128 timeout 300 python tools/profile_ops.py resnet50 256 > gpurun_out/ops_fold128.log 2>&1
timeout 300 python tools/profile_ops.py resnet50 256 > gpurun_out/ops_default.log 2>&1
cat gpurun_out/ab1.log
