cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --import-source on --clock-control none -k regex:chain_gemm -c 1 -o gpurun_out/chain1 python tools/profile_ops.py resnet50 256 > /dev/null 2>&1
