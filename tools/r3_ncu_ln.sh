cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:layernorm_rows --launch-skip 26 --launch-count 1 -o gpurun_out/r3_ln python tools/ncu_target.py bert 128 > /dev/null 2>&1
ncu -i gpurun_out/r3_ln.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"Achieved Occupancy"|"Issued Ipc Active"|"No Eligible"|"L2 Hit Rate"|"DRAM Throughput"|"Memory Throughput"|"Registers Per Thread"'
