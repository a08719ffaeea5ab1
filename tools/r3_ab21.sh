cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py bert 128 >> gpurun_out/ab.txt 2>&1
done
sort -k1,1 -s gpurun_out/ab.txt
python tools/profile_ops.py bert 128 1 2>&1 | grep -m2 layernorm
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:layernorm --launch-skip 26 --launch-count 1 python tools/ncu_target.py bert 128 2>/dev/null | grep -E "layernorm|duration"
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_bert_mask.py -q -rf -x -k bert 2>&1 | tail -3
