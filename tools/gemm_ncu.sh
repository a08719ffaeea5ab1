cd $GRAFT_REPO_ROOT
export B2_DEV=1   # developer knobs (B2_*) honoured
B2_PAIR=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/g1 python tools/gemm_micro.py 12544 2048 512 > /dev/null 2>&1
B2_PAIR=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/g2 python tools/gemm_micro.py 12544 2048 512 > /dev/null 2>&1
B2_PAIR=0 timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/g3 python tools/gemm_micro.py 16384 4096 4096 > /dev/null 2>&1
