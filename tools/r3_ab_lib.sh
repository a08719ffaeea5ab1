# A/B: graph-replayed forwards of the working tree vs ab/libb2_base.so (HEAD), then GPU parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in ${AB_MODELS:-"resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256" "resnet50 16" "resnet50 1"}; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_base.so AB_LABEL=base timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
cat gpurun_out/ab.txt
timeout 300 python tools/det_layers.py bert 128 3 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu.py tests/test_gpu_bert_mask.py -x -q 2>&1 | tail -5
