"""Run-to-run determinism per layer: two forwards of the same batch, every
materialised tensor compared; prints the first ops whose outputs differ.
Knobs from the environment (B2_DEV=1 B2_PAIR=0 ...)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import plan_ref  # noqa: E402
from paper_2006_05096_b200 import plan as P, runtime as R, zoo  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
blob = zoo.build_plan(name, P.DT_BF16)
pl = P.decode(blob)
x = plan_ref.make_inputs(pl, B, 5)
plan = R.Plan(blob, P.DT_BF16)
outs = []
for r in range(reps):
    plan.predict(x)
    snap = {}
    for i, o in enumerate(pl.ops):
        _, dst = plan_ref.op_io(o)
        if dst is None:
            continue
        v = plan.read_tensor(B, dst, pl.tensors[dst].elems, pl.tensors[dst].kind)
        if v is not None:
            snap[i] = (o.name, np.asarray(v))
    outs.append(snap)
label = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("B2_"))
bad = []
for r in range(1, reps):
    for i in sorted(outs[0]):
        a, b = outs[0][i][1], outs[r][i][1]
        if not np.array_equal(a, b):
            rows = np.flatnonzero(np.any(a.reshape(B, -1) != b.reshape(B, -1), axis=1))
            bad.append((r, i, outs[0][i][0], len(rows), rows[:6].tolist()))
            break
print(f"[{label}] {name} b={B}: " + ("deterministic" if not bad else f"FIRST DIFFS {bad}"),
      flush=True)
