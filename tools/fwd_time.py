"""Graph-replayed forward time of one model at one batch (b2_bench, CUDA
events): prints `<label> <model> b=<B> ms=<median of 3 runs of K replays>`.
The label is $AB_LABEL (the B2_* knobs of the run, for A/B matrices)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_05096_b200 import plan as P, runtime as R, zoo  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
K = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dt = P.DT_BF16
plan = R.Plan(zoo.build_plan(name, dt), dt)
plan.bench(B, 3, 2, seed=1)
runs = []
for r in range(3):
    lat, comp = plan.bench(B, K, 5, seed=r)
    runs.append(float(comp[-1]) / K)
print(f"{os.environ.get('AB_LABEL', 'default'):28s} {name} b={B} ms={np.median(runs):.4f} "
      f"runs={[round(x, 4) for x in runs]}", flush=True)
