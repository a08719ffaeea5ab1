"""Where a sweep's non-device time goes: plan creation (decode + weight
upload) and per-batch state (workspaces, tensor maps, graph capture)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_05096_b200 import plan as P, runtime as R, zoo
for name in sys.argv[1].split(","):
    t = time.perf_counter(); blob = zoo.build_plan(name, P.DT_BF16); tb = time.perf_counter() - t
    t = time.perf_counter(); plan = R.Plan(blob, P.DT_BF16); tc = time.perf_counter() - t
    firsts = []
    for b in (1, 16, 256):
        t = time.perf_counter(); plan.bench(b, 1, 0, seed=1); t1 = time.perf_counter() - t
        t = time.perf_counter(); plan.bench(b, 1, 0, seed=1); t2 = time.perf_counter() - t
        firsts.append(f"b{b}: first {t1*1e3:.0f} ms, again {t2*1e3:.1f} ms")
    print(f"{name}: build_plan {tb:.2f} s (host, converter side), Plan() {tc:.2f} s; " + "; ".join(firsts))
    plan.close()
