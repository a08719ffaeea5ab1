# producer rewrite: parity of the GEMM paths + A/B forward times (new vs ab/libb2_base.so = HEAD)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu.py -q -rf -x > gpurun_out/t_ab2.log 2>&1
tail -3 gpurun_out/t_ab2.log
for m in "resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256" "resnet50 1" "resnet50 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab2.log 2>&1
  AB_LABEL=base B2_LIB=ab/libb2_base.so timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab2.log 2>&1
done
cat gpurun_out/ab2.log
B2_PARITY_LOG=gpurun_out/parity_margins.json timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -rf > gpurun_out/fullsize.log 2>&1
tail -3 gpurun_out/fullsize.log
