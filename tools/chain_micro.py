"""Graph-replayed chain of L identical LINEAR layers (M x K -> K): per-layer
device time inside a CUDA graph, free of eager launch overhead."""
import os, sys
os.environ.setdefault("B2_DEV", "1")   # developer knobs (B2_*) honoured
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_05096_b200 import plan as P, runtime as R
M, K, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
b = P.PlanBuilder("chain")
x = b.tensor(K); b.in_elems = K
b.op_p(P.OP_INPUT, [x, K, 1, 1, K])
rng = np.random.default_rng(0)
cur = x
for i in range(L):
    y = b.tensor(K)
    b.op_p(P.OP_LINEAR, [cur, y, b.weight(rng.standard_normal((K, K)) / np.sqrt(K)), b.weight(np.zeros(K)), K, K, 1, 1, -1, K])
    cur = y
b.out_elems = K
b.op_p(P.OP_OUTPUT, [1, cur, 0])
plan = R.Plan(b.build(P.DT_BF16), P.DT_BF16)
plan.bench(M, 3, 2, seed=1)
lat, comp = plan.bench(M, 20, 5, seed=0)
ms = float(np.median(lat))
print(f"chain M={M} K={K} L={L}: {ms*1e3:.1f} us/forward, {ms*1e3/L:.2f} us/layer, {2*M*K*K*L/ms/1e9:.1f} TF/s")
