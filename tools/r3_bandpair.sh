# N = 128 band conv on a CTA pair with streamed weights: parity + A/B against HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out

timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x 2>&1 | tail -4
for rep in 1 2 3; do
for m in "resnet50 256" "resnet50 64"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_bp.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab_bp.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab_bp.txt | grep -v "^ \|Trace\|File"
timeout 300 python tools/profile_ops.py resnet50 256 > gpurun_out/ops_r50_bp.txt 2>&1
grep "28x28x128->28x28x128" gpurun_out/ops_r50_bp.txt
