cd $GRAFT_REPO_ROOT
for rep in 1 2; do for ao in 0 1; do
  B2_ALT_ORDER=$ao timeout 120 python bench.py --no-cpu --no-sweep --steps 50 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('ALT=$ao', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
done; done
timeout 300 python -m pytest tests/test_gpu.py -x -q -k "resnet or invariance" 2>&1 | tail -1
