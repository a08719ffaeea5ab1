"""Per-op device times of one forward (eager, CUDA events between ops)."""
import os, sys, json
os.environ.setdefault("B2_DEV", "1")   # developer knobs (B2_*) honoured
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_05096_b200 import zoo, plan as P, runtime as R
name = sys.argv[1]; B = int(sys.argv[2]); dt = int(sys.argv[3]) if len(sys.argv) > 3 else 1
blob = zoo.build_plan(name, dt)
pl = P.decode(blob)
plan = R.Plan(blob, dt)
prof = plan.profile_ops(B, iters=5)
esz = 2 if dt == 1 else 4
tot = sum(ms for _, ms in prof)
rows = []
for o, (k, ms) in zip(pl.ops, prof):
    fl = 0; by = 0
    if o.kind == P.OP_CONV:
        fl = 2*o[12]*o[13]*o[7]*o[8]*o[9]*o[6]*B
        by = esz*B*(pl.tensors[o[0]].elems + pl.tensors[o[1]].elems*(2 if o[15] >= 0 else 1))
        desc = f"conv {o[4]}x{o[5]}x{o[6]}->{o[12]}x{o[13]}x{o[7]} k{o[8]} s{o[10]}"
    elif o.kind == P.OP_LINEAR:
        fl = 2*o[6]*o[5]*o[4]*B
        by = esz*B*o[6]*(o[4] + o[5]) + esz*o[4]*o[5]
        desc = f"linear M={B*o[6]} K={o[4]} N={o[5]}"
    else:
        desc = o.name
        try:
            by = esz*B*(pl.tensors[o[0]].elems + pl.tensors[o[1]].elems) if o.kind not in (P.OP_OUTPUT, P.OP_TOKENS) else 0
        except IndexError:
            by = 0
    rows.append((ms, desc, fl/ms/1e9 if ms > 0 else 0, by/ms/1e6 if ms > 0 else 0))
print(f"{name} b={B} dtype={dt}: total {tot:.3f} ms over {len(prof)} ops -> {plan.flops_per_sample*B/tot/1e9:.1f} TFLOP/s")
for ms, desc, tf, gbs in rows:
    print(f"  {ms:8.4f} ms {100*ms/tot:5.1f}%  {tf:7.1f} TF/s {gbs:7.0f} GB/s  {desc}")
