cd $GRAFT_REPO_ROOT
for pr in 0 1; do
export B2_PAIR=$pr
for args in "50176 1024 256" "50176 256 1024 res" "12544 2048 512" "12544 512 2048 res" "200704 512 128" "802816 64 256 res" "200704 2048 512" "16384 4096 4096"; do
  timeout 60 python tools/gemm_micro.py $args
done
timeout 60 python tools/conv_micro.py 256 7 7 512 512 3 1
timeout 60 python tools/conv_micro.py 256 14 14 256 256 3 1
done
