cd $GRAFT_REPO_ROOT
for rep in 1 2; do for ch in 0 1; do
  B2_CHAIN=$ch timeout 120 python bench.py --no-cpu --no-sweep --steps 50 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('CHAIN=$ch', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
done; done
