# ncu --set full, one launch each of BERT b=128's attention, LayerNorm and FFN-up GEMM
cd $GRAFT_REPO_ROOT
E=gpurun_out/bf; mkdir -p $E
timeout 600 ncu --set full --clock-control none -k regex:attn_tc -s 2 -c 1 -o $E/attn python tools/ncu_target.py bert 128 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:layernorm_rows -s 2 -c 1 -o $E/ln python tools/ncu_target.py bert 128 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tc_gemm2 -s 6 -c 1 -o $E/ffnup python tools/ncu_target.py bert 128 > /dev/null 2>&1
ls -la $E
