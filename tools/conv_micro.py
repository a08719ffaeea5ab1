"""Micro-benchmark one conv shape through a single-CONV plan (per-op CUDA events)."""
import os, sys
os.environ.setdefault("B2_DEV", "1")   # developer knobs (B2_*) honoured
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_05096_b200 import plan as P, runtime as R
B, H, W, C, Cout, Rk, st = [int(v) for v in sys.argv[1:8]]
pad = Rk // 2
OH = (H + 2 * pad - Rk) // st + 1; OW = (W + 2 * pad - Rk) // st + 1
b = P.PlanBuilder("cmicro")
Cp = max(8, C); x = b.tensor(H, W, Cp); b.in_elems = C * H * W
b.op_p(P.OP_INPUT, [x, C, H, W, Cp])
rng = np.random.default_rng(0)
y = b.tensor(OH, OW, Cout)
b.op_p(P.OP_CONV, [x, y, b.weight(rng.standard_normal((Cout, Rk, Rk, Cp)) * 0.05), b.weight(np.zeros(Cout)), H, W, Cp, Cout, Rk, Rk, st, pad, OH, OW, 1, -1])
b.out_elems = b.tensors[y].elems
b.op_p(P.OP_OUTPUT, [1, y, 0])
plan = R.Plan(b.build(P.DT_BF16), P.DT_BF16)
prof = plan.profile_ops(B, iters=5)
ms = prof[1][1]
fl = 2 * B * OH * OW * Cout * Rk * Rk * C
print(f"conv B={B} {H}x{W}x{C}->{OH}x{OW}x{Cout} k{Rk} s{st} stages={os.environ.get('B2_STAGES','auto')} mode={os.environ.get('B2_EPI_MODE','0')}: {ms*1e3:.1f} us {fl/ms/1e9:.1f} TF/s")
