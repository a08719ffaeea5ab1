cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab.txt 2>&1
done
sort -k2,3 -s gpurun_out/ab.txt
python tools/profile_ops.py resnet50 256 1 > gpurun_out/ops_new.txt 2>&1
B2_LIB=ab/libb2_head.so python tools/profile_ops.py resnet50 256 1 > gpurun_out/ops_head.txt 2>&1
paste <(cut -c1-12 gpurun_out/ops_new.txt) <(cut -c1-80 gpurun_out/ops_head.txt) | head -20; tail -8 gpurun_out/ops_new.txt
timeout 600 python tools/det_layers.py resnet50 256 4 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py -q -rf -x 2>&1 | tail -3
