# round 2, first GPU pass: NVML probe, full-size parity, the whole GPU suite, bench, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 python tools/nvml_probe.py > gpurun_out/nvml_probe.log 2>&1
B2_PARITY_LOG=gpurun_out/parity_margins.json timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/fullsize.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/gputests.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
tail -3 gpurun_out/fullsize.log gpurun_out/gputests.log; cat gpurun_out/bench.json | head -c 1500
