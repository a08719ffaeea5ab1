cd $GRAFT_REPO_ROOT
timeout 60 python tools/conv_micro.py 256 14 14 512 512 3 2
timeout 60 python tools/conv_micro.py 256 28 28 256 256 3 2
timeout 60 python tools/conv_micro.py 256 7 7 512 512 3 1
timeout 60 python tools/conv_micro.py 256 14 14 256 256 3 1
timeout 60 python tools/conv_micro.py 256 14 14 1024 2048 1 2
timeout 60 python tools/conv_micro.py 256 28 28 512 1024 1 2
timeout 120 python bench.py --no-cpu --steps 30 --warmup 5 --no-sweep | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'], d['e2e']['value'])"
