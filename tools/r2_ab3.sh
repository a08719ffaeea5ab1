# chain/band producers: parity + A/B vs ab/libb2_base.so + per-launch ncu metrics
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_conv.py tests/test_gpu.py -q -rf > gpurun_out/t_ab3.log 2>&1
tail -3 gpurun_out/t_ab3.log
for m in "resnet50 256" "bert 128" "vgg16 256" "mobilenet_v2 256"; do
  AB_LABEL=new timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab3.log 2>&1
  AB_LABEL=base B2_LIB=ab/libb2_base.so timeout 300 python tools/fwd_time.py $m >> gpurun_out/ab3.log 2>&1
done
cat gpurun_out/ab3.log
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launch_metrics2.csv python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
B2_PARITY_LOG=gpurun_out/parity_margins.json timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -rf > gpurun_out/fullsize.log 2>&1
tail -3 gpurun_out/fullsize.log
