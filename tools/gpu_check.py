"""Dev check on a GPU box: parity of every model vs the numpy oracle, fp32 and bf16."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2006_05096_b200 import zoo, plan as P, runtime as R
import plan_ref

models = sys.argv[1].split(",") if len(sys.argv) > 1 else ["mlp", "resnet50", "mobilenet_v2", "bert", "vgg16"]
B = int(os.environ.get("B", "2"))
for name in models:
    t0 = time.time()
    blob = zoo.build_plan(name, P.DT_FP32)
    pl = P.decode(blob)
    x = plan_ref.make_inputs(pl, B, 0)
    ref = plan_ref.forward(pl, x)
    print(f"[{name}] plan {len(blob)/1e6:.1f} MB, oracle done {time.time()-t0:.1f}s", flush=True)
    for dt in (P.DT_FP32, P.DT_BF16):
        try:
            plan = R.Plan(blob, dt)
            out = plan.predict(x)
            err = plan_ref.normwise_err(out, ref)
            tol = 1e-4 if dt == P.DT_FP32 else 2e-2
            print(f"  dtype={dt} err={err:.3e} tol={tol} {'OK' if err <= tol else 'FAIL'} finite={np.isfinite(out).all()}", flush=True)
            if name in ("resnet50", "bert", "mlp") and dt == P.DT_BF16:
                for bb in (1, 32, 256 if name != "bert" else 64):
                    lat, comp = plan.bench(bb, n=20, warmup=3)
                    med = float(np.median(lat))
                    print(f"    bench b={bb}: p50 {med:.3f} ms -> {bb/med*1e3:.0f} samples/s, {plan.flops_per_sample*bb/med/1e9:.1f} TFLOP/s", flush=True)
            plan.close()
        except Exception as e:
            print(f"  dtype={dt} EXC {type(e).__name__}: {e}", flush=True)
