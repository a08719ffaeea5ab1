import sys; sys.path[:0]=['oracle','.']
import numpy as np, plan_ref
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
blob = zoo.build_plan('resnet50', P.DT_FP32); pl = P.decode(blob)
x = plan_ref.make_inputs(pl, 2, 11)
plan = R.Plan(blob, P.DT_BF16); plan.predict(x)
rt = lambda t: plan.read_tensor(2, t, pl.tensors[t].elems, pl.tensors[t].kind)
for i, name, e in plan_ref.layerwise_errors(pl, rt, x, True):
    if e > 1e-2: print(i, name, e, pl.ops[i][:16])
print('done')
