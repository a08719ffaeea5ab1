# stream-K CTA-pair GEMM: parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -rf -x -k "bert or resnet" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py tests/test_gpu_bert_mask.py -q -rf -x 2>&1 | tail -4
for rep in 1 2; do
for m in "bert 128" "resnet50 256" "vgg16 256"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_sk.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_sk.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_sk.txt | grep -v "^ \|Trace\|File"
timeout 300 python tools/profile_ops.py bert 128 > gpurun_out/ops_bert_sk.txt 2>&1; sed -n 2,12p gpurun_out/ops_bert_sk.txt
timeout 300 python tools/profile_ops.py resnet50 256 > gpurun_out/ops_r50_sk.txt 2>&1; head -1 gpurun_out/ops_r50_sk.txt
