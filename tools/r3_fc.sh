# small-M linears (classifier heads, BERT pooler): tile width / split-K choices
cd $GRAFT_REPO_ROOT
export B2_DEV=1
for sh in "256 2048 1000" "256 1280 1000" "128 768 768"; do
  for bn in 0 32 64 128 256; do
    echo "bn=$bn $(B2_FORCE_BN=$bn timeout 60 python tools/gemm_micro.py $sh 2>&1 | tail -1)"
  done
  echo "nosplit $(B2_SPLIT=0 timeout 60 python tools/gemm_micro.py $sh 2>&1 | tail -1)"
done
