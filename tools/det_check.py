"""Run-to-run determinism check of one model at one batch (first vs second predict)."""
import os, sys
os.environ.setdefault("B2_DEV", "1")   # developer knobs (B2_*) honoured
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
from oracle import plan_ref
name, batch = sys.argv[1], int(sys.argv[2])
blob = zoo.build_plan(name, P.DT_BF16)
pl = P.decode(blob)
x = plan_ref.make_inputs(pl, batch, 5)
plan = R.Plan(blob, P.DT_BF16)
ys = [plan.predict(x) for _ in range(3)]
bad = [np.flatnonzero(np.any(ys[i] != ys[2], axis=1)) for i in range(2)]
print(name, batch, os.environ.get("B2_PAIR", ""), os.environ.get("B2_PAIR_MIN_K", ""),
      "rows differing run0 vs run2:", len(bad[0]), bad[0][:10], "run1 vs run2:", len(bad[1]))
