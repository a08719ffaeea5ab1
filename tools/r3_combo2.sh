cd $GRAFT_REPO_ROOT
tools/tma_write > gpurun_out/tma_write.txt 2>&1; cat gpurun_out/tma_write.txt
python tools/profile_ops.py bert 128 1 > gpurun_out/ops_bert_new.txt 2>&1
B2_LIB=ab/libb2_base.so python tools/profile_ops.py bert 128 1 > gpurun_out/ops_bert_base.txt 2>&1
grep -m3 attention gpurun_out/ops_bert_new.txt; grep -m3 attention gpurun_out/ops_bert_base.txt
head -1 gpurun_out/ops_bert_new.txt; head -1 gpurun_out/ops_bert_base.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm2_kernel --launch-skip 34 --launch-count 3 \
    -o gpurun_out/r3_expand python tools/ncu_target.py resnet50 256 > gpurun_out/ncu_expand.log 2>&1
