# three default-config bench runs on one box (run-to-run spread of the headline)
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  timeout 900 python bench.py --no-sweep --no-c4 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());c=d['clocks'];print('value %.1f samples/s  ms_per_step %.4f  e2e %.1f  frac %.4f  sm_mhz %s (min %s)  reasons %s  samples %s' % (d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],c['sm_mhz'],c.get('sm_min_mhz'),c['reasons'],c.get('samples')))"
done
