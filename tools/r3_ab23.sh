cd $GRAFT_REPO_ROOT
timeout 300 python tools/det_layers.py bert 128 3 2>&1 | tail -1
for rep in 1 2 3; do
  AB_LABEL=fold timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab.txt 2>&1
  B2_DEV=1 B2_LN_FOLD=0 AB_LABEL=nofold timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab.txt 2>&1
done
sort -k1,1 -s gpurun_out/ab.txt
python tools/profile_ops.py bert 128 1 2>&1 | sed -n 1,10p
B2_PARITY_LOG=gpurun_out/pm.json timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_bert_mask.py -q -rf -k bert 2>&1 | tail -8
