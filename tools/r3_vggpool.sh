# fused 2x2 pool: max on the raw accumulators, bias + ReLU once — parity + A/B on VGG-16
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x -k "vgg or pool" 2>&1 | tail -2
for rep in 1 2 3; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py vgg16 256 >> gpurun_out/ab_vp.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py vgg16 256 >> gpurun_out/ab_vp.txt 2>&1
done
sort -k2,3 -s gpurun_out/ab_vp.txt | grep -v "^ \|Trace\|File"
