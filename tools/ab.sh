cd $GRAFT_REPO_ROOT
for pd in 0 1; do
  export B2_PDL=$pd
  echo "== PDL=$pd"
  timeout 60 python tools/chain_micro.py 18944 256 20
  timeout 60 python tools/chain_micro.py 256 1024 20
  timeout 120 python bench.py --no-cpu --steps 30 --warmup 5 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'], d['e2e']['value'], {k: v['p50_ms'] for k, v in d['per_batch'].items()})"
done
