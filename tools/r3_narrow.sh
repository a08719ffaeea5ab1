cd $GRAFT_REPO_ROOT
export B2_DEV=1
for sh in "3211264 32 16" "3211264 32 64" "802816 64 64" "802816 64 128"; do
  for bn in 32 64 128; do
    B2_FORCE_BN=$bn timeout 120 python tools/gemm_micro.py $sh 2>&1 | tail -1 | sed "s/^/bn=$bn /"
  done
done
