cd $GRAFT_REPO_ROOT
for m in "bert 128" "vgg16 256" "mobilenet_v2 256"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
sort -k2,3 -s gpurun_out/ab.txt
python tools/profile_ops.py vgg16 256 1 2>&1 | sed -n 2,3p
python tools/profile_ops.py bert 128 1 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py -q -rf -x 2>&1 | tail -3
