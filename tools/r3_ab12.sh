cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  AB_LABEL=default timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab.txt 2>&1
  B2_DEV=1 B2_CHAIN_DS2=0 AB_LABEL=nochain_ds2 timeout 300 python tools/fwd_time.py resnet50 256 >> gpurun_out/ab.txt 2>&1
done
sort -k1,1 -s gpurun_out/ab.txt
B2_DEV=1 B2_CHAIN_DS2=0 timeout 300 python tools/profile_ops.py resnet50 256 1 > gpurun_out/ops_r50_nods2.txt 2>&1
timeout 300 python tools/profile_ops.py resnet50 256 1 > gpurun_out/ops_r50.txt 2>&1
head -20 gpurun_out/ops_r50.txt; head -22 gpurun_out/ops_r50_nods2.txt
