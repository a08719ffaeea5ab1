# A/B: baseline build (ab/libb2_base.so, HEAD) vs working tree, same box, interleaved
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lib in ab/libb2_base.so paper_2006_05096_b200/libb2.so; do
  echo "== $lib"
  export B2_LIB=$PWD/$lib
  for args in "12544 2048 512" "12544 512 2048 res" "300 2048 512" "50176 1024 256"; do
    B2_PAIR=0 timeout 60 python tools/gemm_micro.py $args
  done
  timeout 60 python tools/conv_micro.py 256 7 7 512 512 3 1
  timeout 60 python tools/conv_micro.py 4 7 7 512 512 3 1
done
done
