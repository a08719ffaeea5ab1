cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for m in "bert 128" "resnet50 256" "mobilenet_v2 256"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_base.so AB_LABEL=base timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab.txt
python tools/profile_ops.py bert 128 1 > gpurun_out/ops_bert_new.txt 2>&1; sed -n 1,10p gpurun_out/ops_bert_new.txt
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -4
