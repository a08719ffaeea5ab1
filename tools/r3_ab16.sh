cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for m in "resnet50 1" "resnet50 16" "bert 1" "mobilenet_v2 1" "resnet50 256"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab.txt
timeout 2400 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -3
