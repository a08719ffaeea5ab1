# attention softmax: two max chains, packed scale-shift and row sum
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_bert_mask.py -q -rf -x -k "bert or attention or mask" 2>&1 | tail -2
for rep in 1 2 3 4; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_at3.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_at3.txt 2>&1
done
sort -k2,3 -s gpurun_out/ab_at3.txt | grep -v "^ \|Trace\|File"
timeout 300 python tools/profile_ops.py bert 128 2>&1 | grep attention | head -3
B2_LIB=ab/libb2_head.so timeout 300 python tools/profile_ops.py bert 128 2>&1 | grep attention | head -3
