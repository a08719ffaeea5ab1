# BERT GEMMs: single-CTA vs CTA-pair kernels
cd $GRAFT_REPO_ROOT
for s in "16384 768 3072" "16384 768 2304" "16384 768 768" "16384 3072 768" "50176 256 1024" "12544 4608 512" "12544 512 2048"; do
 python tools/gemm_micro.py $s; B2_PAIR_MIN_K=64 B2_PAIR_MIN_M=1 python tools/gemm_micro.py $s; B2_PAIR=0 python tools/gemm_micro.py $s; done
