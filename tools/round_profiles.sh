# Refresh the committed measurement evidence: bench line, ncu launch list of one
# ResNet-50 b=256 forward (+ DRAM bytes), and the C4 sweep on one GPU.
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
timeout 900 python tools/sweep_bench.py gpurun_out/sweep_c4 > gpurun_out/sweep.log 2>&1
