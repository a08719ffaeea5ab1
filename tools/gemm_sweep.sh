cd $GRAFT_REPO_ROOT
export B2_DEV=1   # developer knobs (B2_*) honoured
for sk in 0 1; do
export B2_SPLIT=$sk
for args in "12544 2048 512" "12544 512 2048 res" "50176 1024 256" "300 2048 512"; do
  timeout 60 python tools/gemm_micro.py $args
done
timeout 60 python tools/conv_micro.py 256 7 7 512 512 3 1
timeout 60 python tools/conv_micro.py 1 7 7 512 512 3 1
timeout 60 python tools/conv_micro.py 256 14 14 512 512 3 2
done
