cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# second forward of the eager pass: 48 tc_gemm2 per forward; QKV, O-proj, FFN-up, FFN-down per layer
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm2_kernel --launch-skip 52 --launch-count 4 \
    -o gpurun_out/r3_bert_gemm python tools/ncu_target.py bert 128 > gpurun_out/ncu_bert_gemm.log 2>&1; echo rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:layernorm --launch-skip 26 --launch-count 1 \
    -o gpurun_out/r3_bert_ln python tools/ncu_target.py bert 128 > gpurun_out/ncu_bert_ln.log 2>&1; echo rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc --launch-skip 13 --launch-count 1 \
    -o gpurun_out/r3_bert_attn python tools/ncu_target.py bert 128 > gpurun_out/ncu_bert_attn.log 2>&1; echo rc=$?
