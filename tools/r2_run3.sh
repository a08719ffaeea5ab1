# GPU pass: full-size parity with per-op bounds, daemon tests, controller-driven C4 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B2_PARITY_LOG=gpurun_out/parity_margins.json timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -rf > gpurun_out/fullsize.log 2>&1
timeout 900 python -m pytest tests/test_gpu_daemon.py -q -s -rf > gpurun_out/daemon.log 2>&1
timeout 900 python tools/sweep_bench.py gpurun_out/r2_sweep_c4_ctrl > gpurun_out/sweep_ctrl.log 2>&1
tail -3 gpurun_out/fullsize.log; tail -15 gpurun_out/daemon.log; tail -3 gpurun_out/sweep_ctrl.log
