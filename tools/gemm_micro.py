"""Micro-benchmark one GEMM shape through a single-LINEAR plan (per-op CUDA events)."""
import os, sys
os.environ.setdefault("B2_DEV", "1")   # developer knobs (B2_*) honoured
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_05096_b200 import plan as P, runtime as R
M, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
res = len(sys.argv) > 4 and sys.argv[4] == "res"
b = P.PlanBuilder("micro")
x = b.tensor(K); b.in_elems = K
b.op_p(P.OP_INPUT, [x, K, 1, 1, K])
rng = np.random.default_rng(0)
r = -1
if res:
    r = b.tensor(N)
    b.op_p(P.OP_LINEAR, [x, r, b.weight(rng.standard_normal((N, K)) * 0.1), b.weight(np.zeros(N)), K, N, 1, 0, -1, K])
y = b.tensor(N)
ACT = int(os.environ.get("MICRO_ACT", 1))   # 0 none, 1 relu, 2 relu6, 3 gelu, 4 tanh
b.op_p(P.OP_LINEAR, [x, y, b.weight(rng.standard_normal((N, K)) * 0.1), b.weight(np.zeros(N)), K, N, 1, ACT, r, K])
b.out_elems = b.tensors[y].elems
b.op_p(P.OP_OUTPUT, [1, b.tensor(1) if False else y, 0])
DT = int(os.environ.get("MICRO_DTYPE", P.DT_BF16))
blob = b.build(P.DT_BF16)
plan = R.Plan(blob, DT)
prof = plan.profile_ops(M, iters=5)
ms = prof[-2][1]
byts = (2 if DT == P.DT_BF16 else 4) * M * (K + N * (2 if res else 1))
print(f"M={M} K={K} N={N} res={res} mode={os.environ.get('B2_EPI_MODE','0')} stages={os.environ.get('B2_STAGES','auto')}: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TF/s  {byts/ms/1e6:.0f} GB/s")
