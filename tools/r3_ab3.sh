cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for m in "bert 128" "resnet50 256" "mobilenet_v2 256" "resnet50 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_base.so AB_LABEL=base timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu.py tests/test_gpu_bert_mask.py -q 2>&1 | tail -3
timeout 1800 python -m pytest tests/test_gpu_sanitize.py -q -rf 2>&1 | tail -8
