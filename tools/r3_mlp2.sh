cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mlp2 -c 1 -o gpurun_out/r3_mlp2 python tools/ncu_target.py mlp 16 > gpurun_out/ncu_mlp.log 2>&1
ncu -i gpurun_out/r3_mlp2.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"Registers Per Thread"'
