"""compute-sanitizer target: one forward (plus the eager per-op pass, which
launches every kernel outside a CUDA graph) of a model at a small batch.

    compute-sanitizer --tool memcheck python tools/sanitize_target.py resnet50 16
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import plan_ref  # noqa: E402
from paper_2006_05096_b200 import plan as P, runtime as R, zoo  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
dt = int(sys.argv[3]) if len(sys.argv) > 3 else P.DT_BF16
blob = zoo.build_plan(name, dt)
pl = P.decode(blob)
plan = R.Plan(blob, dt)
y = plan.predict(plan_ref.make_inputs(pl, B, 0))
plan.profile_ops(B, iters=1)
plan.close()
print("sanitize-target ok", name, B, y.shape)
