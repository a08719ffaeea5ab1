cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/elastic_c5.py gpurun_out/r2_c5 > gpurun_out/c5.log 2>&1
tail -5 gpurun_out/c5.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json;d=json.loads(open('gpurun_out/bench.json').read());s=d['sweep_c4'];print(d['value'],d['ms_per_step'],d['e2e']['value'],s['wall_s'],s['busiest_rank_device_s'])"
tail -3 gpurun_out/bench.err
