cd $GRAFT_REPO_ROOT
for m in "mlp 1" "mlp 16" "mlp 64"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_base.so AB_LABEL=base timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
for rep in 1 2; do
for m in "bert 128" "bert 8"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab.txt
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_bert_mask.py -q -rf -x 2>&1 | tail -4
python tools/profile_ops.py bert 128 1 > gpurun_out/ops_bert_new.txt 2>&1; sed -n 1,10p gpurun_out/ops_bert_new.txt
