cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -k "split" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu.py -x -q 2>&1 | tail -1
for sk in 0 1; do
  B2_SPLIT=$sk timeout 200 python bench.py --no-cpu --steps 30 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('SPLIT=$sk', d['ms_per_step'], {k: v['p50_ms'] for k, v in d['per_batch'].items()})"
done
