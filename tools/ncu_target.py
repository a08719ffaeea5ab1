"""Small driver for ncu captures: one eager forward (plus warm-up) of a model."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_05096_b200 import zoo, plan as P, runtime as R
name = sys.argv[1]; B = int(sys.argv[2]); dt = int(sys.argv[3]) if len(sys.argv) > 3 else 1
plan = R.Plan(zoo.build_plan(name, dt), dt)
plan.profile_ops(B, iters=1)
print("done")
