# ReLU / ReLU6 on packed bf16 after the pack: parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py tests/test_gpu_bert_mask.py -q -rf -x 2>&1 | tail -2
for rep in 1 2 3; do
for m in "resnet50 256" "vgg16 256" "mobilenet_v2 256" "bert 128"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_f2c.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_f2c.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_f2c.txt | grep -v "^ \|Trace\|File"
