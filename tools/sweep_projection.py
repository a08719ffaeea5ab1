"""Projected C4 sweep wall time on k GPUs from a measured one-GPU controller
sweep (profiles/r3_sweep_c4.json): request-sharded heavy cells (the
sweeprun.plan_shards rule: a cell above half the ideal per-GPU load is split
into k shards, each shard repeating the 10 warm-up requests) and the
setup-aware LPT of sweeprun.lpt_partition (a model's worker start paid once per
GPU hosting it).  Labelled a projection: only one GPU was measured.
usage: sweep_projection.py [sweep.json]"""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2006_05096_b200.sweeprun import lpt_partition  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else "profiles/r3_sweep_c4.json"
d = json.loads(Path(src).read_text())
req, warm = d["requests_per_cell"], d["warmup_requests"]
models = sorted({c["model"] for c in d["cells"]})
start = d["worker_prewarm_s"] / len(models)           # per (model, GPU) worker start
# the controller's wall beyond device time and starts, spread per cell
dev_total = sum(c["device_s"] for c in d["cells"])
over = max(0.0, d["controller_run_s"] - dev_total) / len(d["cells"])
out = {"source": src, "measured_1gpu_wall_s": d["sweep_wall_s_measured"],
       "device_s_total": round(dev_total, 3), "start_s_per_model_gpu": round(start, 3),
       "overhead_s_per_cell": round(over, 4), "projected_wall_s": {}, "shards": {}}
for k in (1, 2, 4, 8):
    total = dev_total + over * len(d["cells"])
    bound = 0.5 * total / k
    units = []
    for c in d["cells"]:
        cost = c["device_s"] + over
        n = 1
        if k > 1 and cost > bound:
            n = min(k, req // 10, math.ceil(cost / bound))
        per_req = c["device_s"] / (req + warm)
        for i in range(n):   # each shard: its share of the timed requests + the full warm-up
            units.append({"model": c["model"], "cost": per_req * (req / n + warm) + over,
                          "cell": f'{c["model"]}:{c["batch"]}', "n": n})
        if n > 1:
            out["shards"].setdefault(str(k), {})[f'{c["model"]}:{c["batch"]}'] = n
    bins = lpt_partition(units, lambda u: u["cost"], k, group=lambda u: u["model"],
                         setup=lambda m: start)
    loads = [sum(u["cost"] for u in b) + start * len({u["model"] for u in b}) for b in bins]
    out["projected_wall_s"][str(k)] = round(max(loads), 3)
p1 = out["projected_wall_s"]["1"]
out["projected_speedup"] = {k: round(p1 / v, 2) for k, v in out["projected_wall_s"].items()}
print(json.dumps(out, indent=1))
