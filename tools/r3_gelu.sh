# GELU in its even form (no sign transfer): parity + A/B against HEAD on BERT
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_bert_mask.py -q -rf -x -k "bert or gelu" 2>&1 | tail -2
for rep in 1 2 3 4; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_gelu.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab_gelu.txt 2>&1
done
sort -k2,3 -s gpurun_out/ab_gelu.txt | grep -v "^ \|Trace\|File"
for i in 1 2; do
  MICRO_ACT=3 timeout 120 python tools/gemm_micro.py 16384 768 3072 2>&1 | tail -1 | sed "s/^/new  /"
  B2_LIB=ab/libb2_head.so MICRO_ACT=3 timeout 120 python tools/gemm_micro.py 16384 768 3072 2>&1 | tail -1 | sed "s/^/head /"
done
