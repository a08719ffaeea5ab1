"""Layerwise oracle check of one model at a dtype; prints ops over tolerance."""
import sys
sys.path[:0] = ['oracle', '.']
import numpy as np, plan_ref
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
name, dt = sys.argv[1], int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 2
tol = 1e-2 if dt == P.DT_BF16 else 1e-5
blob = zoo.build_plan(name, P.DT_FP32); pl = P.decode(blob)
x = plan_ref.make_inputs(pl, B, 11)
plan = R.Plan(blob, dt); out = plan.predict(x)
print('e2e', plan_ref.normwise_err(out, plan_ref.forward(pl, x)))
rt = lambda t: plan.read_tensor(B, t, pl.tensors[t].elems, pl.tensors[t].kind)
errs = plan_ref.layerwise_errors(pl, rt, x, dt == P.DT_BF16)
for i, nm, e in errs:
    if e > tol: print(i, nm, e, pl.ops[i][:16])
print('max', max(e for _, _, e in errs))
