# ncu evidence for ResNet-50 b=256: per-launch tensor/DRAM/xbar table + full set of every tc_gemm2<256>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launch_metrics.csv python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:tc_gemm2_kernel -c 29 -o gpurun_out/r2_full_gemm2 python tools/ncu_target.py resnet50 256 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
