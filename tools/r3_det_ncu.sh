# determinism per layer under the kernel-selection configs + ncu launch tables (default, B2_RES_TMA=0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "B2_DEV=1 B2_PAIR=0 B2_SPLIT=0" "B2_DEV=1 B2_RES_TMA=0 B2_PAIR=0 B2_SPLIT=0"; do
  echo "== $cfg" >> gpurun_out/det.log
  env $cfg timeout 300 python tools/det_layers.py resnet50 256 4 >> gpurun_out/det.log 2>&1
done
cat gpurun_out/det.log
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r3_lm_new.csv python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
B2_DEV=1 B2_RES_TMA=0 timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r3_lm_old.csv python tools/ncu_target.py resnet50 256 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r3_lm_bert.csv python tools/ncu_target.py bert 128 > /dev/null 2>&1
ls gpurun_out
