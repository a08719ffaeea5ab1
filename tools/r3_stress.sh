# repeat the determinism / full-size parity tests to catch intermittent failures
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_fullsize.py -q -rf -x 2>&1 | tail -1
done
