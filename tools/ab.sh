cd $GRAFT_REPO_ROOT
for rep in 1 2; do for lib in ab/libb2_base.so paper_2006_05096_b200/libb2.so; do
  B2_LIB=$PWD/$lib timeout 120 python bench.py --no-cpu --no-sweep --steps 50 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
done; done
