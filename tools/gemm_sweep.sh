cd $GRAFT_REPO_ROOT
for pf in 0 1; do
export B2_L2_PREFETCH=$pf
for args in "50176 1024 256" "50176 256 1024 res" "12544 2048 512" "12544 512 2048 res" "200704 512 128" "802816 64 256 res" "802816 256 64"; do
  timeout 60 python tools/gemm_micro.py $args
done
done
