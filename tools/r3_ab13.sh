cd $GRAFT_REPO_ROOT
cat > /tmp/fwd32.py <<'PY'
import os, sys
import numpy as np
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
name, B = sys.argv[1], int(sys.argv[2])
plan = R.Plan(zoo.build_plan(name, P.DT_FP32), P.DT_FP32)
plan.bench(B, 3, 2, seed=1)
runs = []
for r in range(3):
    lat, comp = plan.bench(B, 20, 3, seed=r)
    runs.append(float(comp[-1]) / 20)
print(f"{os.environ.get('AB_LABEL','x'):10s} fp32 {name} b={B} ms={np.median(runs):.4f}", flush=True)
PY
for m in "resnet50 64" "vgg16 16" "mobilenet_v2 64"; do
  AB_LABEL=new timeout 300 python /tmp/fwd32.py $m
  B2_LIB=ab/libb2_head.so AB_LABEL=head timeout 300 python /tmp/fwd32.py $m
done
timeout 1500 python -m pytest tests/test_gpu.py -q -rf -k "parity" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -rf 2>&1 | tail -3
