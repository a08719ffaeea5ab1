cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mlp2 -c 2 -o gpurun_out/r3_mlp python tools/ncu_target.py mlp 64 > gpurun_out/ncu_mlp.log 2>&1
ncu -i gpurun_out/r3_mlp.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"Registers Per Thread"|"Achieved Occupancy"' 
B2_DEV=1 B2_MLP_FUSE=0 timeout 300 ncu --metrics gpu__time_duration.sum --csv python tools/ncu_target.py mlp 64 2>/dev/null | grep -o '"[a-z_0-9]*kernel[^"]*","[^"]*","[^"]*","gpu__time_duration.sum","[^"]*","[0-9.,]*"' | head
