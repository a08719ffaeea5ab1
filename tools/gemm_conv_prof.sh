# ncu --set full of single conv shapes on the tc_gemm path (top-3 late-layer shapes)
cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/l4_3x3 python tools/conv_micro.py 256 7 7 512 512 3 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/l3_1x1a python tools/conv_micro.py 256 14 14 1024 256 1 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o gpurun_out/l1_1x1 python tools/conv_micro.py 256 56 56 256 64 1 1 > /dev/null 2>&1
