cd $GRAFT_REPO_ROOT
export B2_DEV=1
for sh in "3211264 32 16" "802816 64 64" "802816 64 128" "3211264 16 96"; do
  timeout 120 python tools/gemm_micro.py $sh 2>&1 | tail -1 | sed "s/^/bres /"
  B2_BRES=0 timeout 120 python tools/gemm_micro.py $sh 2>&1 | tail -1 | sed "s/^/nobres /"
done
unset B2_DEV
for rep in 1 2; do
for m in "mobilenet_v2 256" "resnet50 256" "resnet50 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab.txt
timeout 1500 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x 2>&1 | tail -3
