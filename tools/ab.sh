cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none -k regex:dwconv3 -c 3 -o gpurun_out/dw python tools/profile_ops.py mobilenet_v2 256 > /dev/null 2>&1
