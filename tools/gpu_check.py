"""Dev check on a GPU box: end-to-end + layerwise parity of every model vs the numpy oracle."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2006_05096_b200 import zoo, plan as P, runtime as R
import plan_ref

models = sys.argv[1].split(",") if len(sys.argv) > 1 else ["mlp", "resnet50", "mobilenet_v2", "bert", "vgg16"]
dts = [int(d) for d in os.environ.get("DTS", "0,1").split(",")]
B = int(os.environ.get("B", "2"))
for name in models:
    t0 = time.time()
    blob = zoo.build_plan(name, P.DT_FP32)
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, B, 0)
    ref = plan_ref.forward(pl, x)
    emu = plan_ref.forward(pl, x, emulate_bf16=True) if 1 in dts else None
    print(f"[{name}] plan {len(blob)/1e6:.1f} MB, oracle done {time.time()-t0:.1f}s", flush=True)
    for dt in dts:
        try:
            plan = R.Plan(blob, dt)
            out = plan.predict(x)
            err = plan_ref.normwise_err(out, ref)
            extra = f" err_vs_bf16emu={plan_ref.normwise_err(out, emu):.3e}" if dt == P.DT_BF16 else ""
            print(f"  dtype={dt} e2e err={err:.3e} finite={np.isfinite(out).all()}{extra}", flush=True)
            rt = lambda t: plan.read_tensor(B, t, pl.tensors[t].elems, pl.tensors[t].kind)
            lw = plan_ref.layerwise_errors(pl, rt, x, emulate_bf16=(dt == P.DT_BF16))
            worst = sorted(lw, key=lambda r: -r[2])[:4]
            tol = 1e-2 if dt == P.DT_BF16 else 1e-5
            bad = [r for r in lw if not (r[2] <= tol)]
            print(f"  layerwise: {len(lw)} ops, worst {[(i, n, f'{e:.2e}') for i, n, e in worst]} -> {'OK' if not bad else 'FAIL ' + str(bad[:5])}", flush=True)
            plan.close()
        except Exception as e:
            import traceback; traceback.print_exc()
            print(f"  dtype={dt} EXC {type(e).__name__}: {e}", flush=True)
