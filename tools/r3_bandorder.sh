# band-major unit order in conv_band_kernel: parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x 2>&1 | tail -4
for rep in 1 2; do
for m in "resnet50 256" "vgg16 256" "mobilenet_v2 256" "resnet50 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_bo.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_bo.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_bo.txt | grep -v "^ \|Trace\|File"
timeout 300 python tools/profile_ops.py resnet50 256 > gpurun_out/ops_r50_bo.txt 2>&1
grep "k3 s1" gpurun_out/ops_r50_bo.txt
