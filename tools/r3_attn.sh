# attention: Q|K and V on separate load barriers — parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_bert_mask.py tests/test_gpu_fullsize.py -q -rf -x -k "bert" 2>&1 | tail -2
for rep in 1 2 3; do
for m in "bert 128" "bert 8"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_at.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_at.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_at.txt | grep -v "^ \|Trace\|File"
timeout 300 python tools/profile_ops.py bert 128 2>&1 | grep attention | head -4
B2_LIB=ab/libb2_head.so timeout 300 python tools/profile_ops.py bert 128 2>&1 | grep attention | head -4
