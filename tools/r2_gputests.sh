# GPU test pass: full-size parity (margins logged) + the whole -m gpu suite, no -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B2_PARITY_LOG=gpurun_out/parity_margins.json timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -s -rf > gpurun_out/fullsize.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf --deselect tests/test_gpu_fullsize.py > gpurun_out/gputests.log 2>&1
tail -5 gpurun_out/fullsize.log; tail -8 gpurun_out/gputests.log
