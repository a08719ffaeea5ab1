cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for m in "bert 128" "bert 16"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab.txt 2>&1
done
done
sort -k2,3 -s gpurun_out/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:layernorm -c 4 --csv python tools/ncu_target.py bert 128 2>/dev/null | grep -o '"layernorm[^"]*".*gpu__time_duration.sum","[^"]*","[0-9.]*"' | tail -2
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py tests/test_gpu_bert_mask.py -q -rf -x -k "bert" 2>&1 | tail -3
