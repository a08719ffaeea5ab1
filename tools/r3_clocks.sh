cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-c4 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['clocks']);print(d['value'],d['ms_per_step'],d['e2e']['value'])"
nvidia-smi --query-gpu=index,pci.bus_id --format=csv; echo CVD=$CUDA_VISIBLE_DEVICES
