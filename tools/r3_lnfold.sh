# LayerNorm fold (BERT output LN -> next QKV / O-projection): parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_bert_mask.py tests/test_gpu_fullsize.py -q -rf -x -k "bert" 2>&1 | tail -4
for rep in 1 2; do
for m in "bert 128" "bert 8"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_ln.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_ln.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_ln.txt | grep -v "^ \|Trace\|File"
timeout 300 python tools/profile_ops.py bert 128 > gpurun_out/ops_bert_lnfold.txt 2>&1; head -12 gpurun_out/ops_bert_lnfold.txt
