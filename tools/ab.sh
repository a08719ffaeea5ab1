cd $GRAFT_REPO_ROOT
for fk in 256 512 1024; do
  export B2_FOLD_MAX_K=$fk
  timeout 60 python tools/gemm_micro.py 12544 512 2048 res
  timeout 60 python tools/gemm_micro.py 3136 512 2048 res
done
