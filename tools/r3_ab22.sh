cd $GRAFT_REPO_ROOT
timeout 600 python tools/det_layers.py resnet50 256 3 2>&1 | tail -1
for rep in 1 2 3; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab.txt 2>&1
done
sort -k1,1 -s gpurun_out/ab.txt
python tools/profile_ops.py resnet50 256 1 2>&1 | grep "k1 s1" | head -12
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_conv.py -q -rf -x 2>&1 | tail -3
