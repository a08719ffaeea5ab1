"""C4 profile sweep on this box through the product path (BASELINE configs[3]):
register -> convert (b200 plugins) -> device-timed cells (n=100, warmup=10)
on b200 workers -> reference CSV.

``--mode controller`` (default): the daemon path — one pool job per model
(devices ["gpu:*"]), heavy cells request-sharded over the GPUs, the
idle-aware Controller granting cells/shards to GPUs from NVML snapshots with
self-load exclusion (sweeprun.ControllerSweep + CellRunner over
Profiler.run_unit; JobStore persistence), one long-lived worker per (model,
GPU).  ``--mode serial``: Profiler.run_sweep model after model on gpu:0 (the
reference's library path).

Writes <out>.csv (the reference profile-table schema) and <out>.json: sweep
wall time on the GPUs used, per-cell device time, the controller's action
log, and a setup-aware LPT projection of the same cells onto 2/4/8 GPUs
(labelled "projected": measured cell times + measured per-worker start).

    python tools/sweep_bench.py profiles/r2_sweep_c4 [--models resnet50,...] [--batches 1,2,...]
"""
import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2006_05096_b200 import converter, toyformat, zoo  # noqa: E402
from paper_2006_05096_b200.dispatcher import Dispatcher, b200_template  # noqa: E402
from paper_2006_05096_b200.hub import Hub, TensorSpec  # noqa: E402
from paper_2006_05096_b200.profiler import results_to_csv  # noqa: E402
from paper_2006_05096_b200.profiler.sweep import JobStore, Profiler  # noqa: E402
from paper_2006_05096_b200.profiler.types import ProfilingJob, SweepSpec  # noqa: E402
from paper_2006_05096_b200.sweeprun import (CellRunner, ControllerSweep, cell_cost,  # noqa: E402
                                            lpt_partition, nvml_hooks, plan_shards)
from paper_2006_05096_b200.telemetry import NvmlProvider, Telemetry  # noqa: E402


def register(hub: Hub, name: str):
    if name == "mlp":
        rec = hub.register("mlp", "toy", toyformat.canonical_json(zoo.make_mlp_graph(0)),
                           [TensorSpec("x", [-1, 784])])
        src = "toy"
    elif name == "bert":
        rec = hub.register("bert", "transformers-bert",
                           converter.pack_bert(zoo.make_torch_model("bert", 0)),
                           [TensorSpec("input_ids", [-1, 128]),
                            TensorSpec("attention_mask", [-1, 128])])
        src = "transformers-bert"
    else:
        rec = hub.register(name, "torchvision",
                           converter.pack_torchvision(zoo.make_torch_model(name, 0), name),
                           [TensorSpec("x", [-1, 3, 224, 224])])
        src = "torchvision"
    plugin = [p for p in converter.b200_plugins((src,)) if p.target_format == "b200-bf16"][0]
    return rec, hub.convert(rec, plugin)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--models", default="mlp,mobilenet_v2,resnet50,bert,vgg16")
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--requests", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--mode", choices=["controller", "serial"], default="controller")
    ap.add_argument("--gpus", type=int, default=0, help="GPUs to use (0 = all visible)")
    args = ap.parse_args()
    if args.mode == "controller":
        return controller_sweep(args)
    models = args.models.split(",")
    batches = [int(b) for b in args.batches.split(",")]
    hub = Hub()
    t0 = time.perf_counter()
    variants = {m: register(hub, m) for m in models}
    convert_s = time.perf_counter() - t0
    tel = Telemetry(NvmlProvider())
    tel.sample_devices()
    work = Path(tempfile.mkdtemp(prefix="b2sweep_"))
    disp = Dispatcher(hub, {"b200": b200_template()}, work, tel.device_ids)
    tel.instance_pid_resolver = disp.pid_of
    tel.instance_device_resolver = disp.device_of
    prof = Profiler(hub, disp, tel, JobStore(hub.store))
    rows, cells, per_model = [], [], {}
    t_sweep = time.perf_counter()
    # long-lived workers, started concurrently (process start, CUDA context and
    # weight upload of the five models overlap instead of running in series)
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(len(models)) as ex:
        futs = {m: ex.submit(disp.dispatch, variants[m][1], "gpu:0", "b200", "grpc-style")
                for m in models}
        warm = {m: f.result() for m, f in futs.items()}
    prewarm_s = time.perf_counter() - t_sweep
    try:
        for m in models:
            rec, var = variants[m]
            job = ProfilingJob(f"c4-{m}", rec.id, var.id,
                               SweepSpec(batch_sizes=batches, devices=["gpu:0"], backends=["b200"],
                                         protocols=["grpc-style"],
                                         requests_per_cell=args.requests,
                                         warmup_requests=args.warmup))
            tm = time.perf_counter()
            res = prof.run_sweep(job, instance=warm[m])
            per_model[m] = {"wall_s": round(time.perf_counter() - tm, 3),
                            "failed_cells": list(job.failed_cells)}
            rows += res
            for r in res:
                # device time of the cell's timed requests (+ warm-up at the same rate)
                dev_s = (args.requests + args.warmup) * r.p50_latency_ms / 1e3
                cells.append({"model": m, "batch": r.batch_size,
                              "samples_s": round(r.peak_throughput, 1),
                              "p50_ms": round(r.p50_latency_ms, 4),
                              "p99_ms": round(r.p99_latency_ms, 4), "device_s": dev_s})
    finally:
        disp.shutdown()
    wall = time.perf_counter() - t_sweep
    # per-model worker start on a GPU (its share of the concurrent pre-warm) is
    # paid once per GPU hosting the model; the rest of the model's non-device
    # wall time (per-batch state + graph capture, RPC) is per cell and moves
    # with the cell
    start = {m: prewarm_s / len(models) for m in models}
    for m in models:
        mc = [c for c in cells if c["model"] == m]
        extra = max(0.0, per_model[m]["wall_s"] - sum(c["device_s"] for c in mc))
        for c in mc:
            c["overhead_s"] = round(extra / len(mc), 4)
    proj = {}
    for k in (1, 2, 4, 8):
        bins = lpt_partition(cells, lambda c: c["device_s"] + c["overhead_s"], k,
                             group=lambda c: c["model"], setup=lambda m: start[m])
        loads = [sum(c["device_s"] + c["overhead_s"] for c in b) +
                 sum(start[m] for m in {c["model"] for c in b}) for b in bins]
        proj[str(k)] = round(max(loads), 3)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.with_suffix(".csv").write_text(results_to_csv(rows))
    summary = {"config": "C4: " + ",".join(models) + " x batches " + args.batches,
               "requests_per_cell": args.requests, "warmup_requests": args.warmup,
               "gpus_measured": 1, "sweep_wall_s_measured": round(wall, 3),
               "convert_s": round(convert_s, 3), "worker_prewarm_s": round(prewarm_s, 3),
               "per_model": per_model,
               "sweep_wall_s_projected_lpt": proj,
               "projection": "setup-aware LPT over measured per-cell device time + per-cell "
                             "overhead (the model's measured wall - device time, split over its "
                             "cells) + one worker start per (model, GPU hosting it)",
               "cells": cells}
    out.with_suffix(".json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: summary[k] for k in ("sweep_wall_s_measured", "sweep_wall_s_projected_lpt",
                                               "per_model")}))
    return 0


def controller_sweep(args) -> int:
    from paper_2006_05096_b200 import plan as P
    from paper_2006_05096_b200.controller import ControllerConfig
    models = args.models.split(",")
    batches = [int(b) for b in args.batches.split(",")]
    hub = Hub()
    t0 = time.perf_counter()
    variants = {m: register(hub, m) for m in models}
    convert_s = time.perf_counter() - t0
    flops = {m: P.flops_per_sample(P.decode(hub.get_blob(variants[m][1].blob_digest)))
             for m in models}
    prov = NvmlProvider()
    tel = Telemetry(prov)
    tel.sample_devices()
    devices = tel.device_ids()[:args.gpus or None]
    work = Path(tempfile.mkdtemp(prefix="b2sweep_"))
    disp = Dispatcher(hub, {"b200": b200_template()}, work, tel.device_ids)
    tel.instance_pid_resolver = disp.pid_of
    tel.instance_device_resolver = disp.device_of
    store = JobStore(hub.store)
    events = []
    prof = Profiler(hub, disp, tel, store,
                    on_event=lambda k, p: events.append((round(time.perf_counter() - t0, 4), k,
                                                         p.get("cell") or p.get("shard"))))
    jobs = [ProfilingJob(f"c4-{m}", variants[m][0].id, variants[m][1].id,
                         SweepSpec(batch_sizes=batches, devices=["gpu:*"], backends=["b200"],
                                   protocols=["grpc-style"], requests_per_cell=args.requests,
                                   warmup_requests=args.warmup)) for m in models]
    model_of = {j.id: m for j, m in zip(jobs, models)}
    cost = lambda j, c: cell_cost(flops[model_of[j.id]], c, c.shard_requests(args.requests),
                                  args.warmup)
    shards = plan_shards(jobs, len(devices), cost)
    for j in jobs:
        store.save(j)
    runner = CellRunner(prof)
    sample, ours_only = nvml_hooks(prov, runner, disp.pid_of)
    t_sweep = time.perf_counter()
    # one worker per (model, GPU), started concurrently before the first grant
    pairs = [(j, j.sweep.cells()[0].on(d)) for j in jobs for d in devices]
    runner.prewarm(pairs)
    prewarm_s = time.perf_counter() - t_sweep
    sweep = ControllerSweep(devices, runner, sample=sample, ours_only=ours_only, quiet_s=0.25,
                            cost_fn=cost, jobs_store=store,
                            config=ControllerConfig(max_cells_per_job=None, order="lpt",
                                                    consecutive_samples=1))
    try:
        run_s = sweep.run(jobs, timeout_s=1800)
    finally:
        runner.shutdown()
        disp.shutdown()
    wall = time.perf_counter() - t_sweep
    rows = [r for j in jobs for r in j.results]
    cells = [{"model": model_of[j.id], "batch": r.batch_size, "device": r.device,
              "samples_s": round(r.peak_throughput, 1), "p50_ms": round(r.p50_latency_ms, 4),
              "p99_ms": round(r.p99_latency_ms, 4),
              "device_s": (args.requests + args.warmup) * r.p50_latency_ms / 1e3}
             for j in jobs for r in j.results]
    per_dev = {}
    for t, a in sweep.actions:
        if a["kind"] == "start_cell":
            per_dev[a["device"]] = per_dev.get(a["device"], 0) + 1
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.with_suffix(".csv").write_text(results_to_csv(rows))
    summary = {"config": "C4: " + ",".join(models) + " x batches " + args.batches,
               "mode": "controller (ControllerSweep + CellRunner, NVML snapshots, self-load "
                       "exclusion, request shards, JobStore)",
               "requests_per_cell": args.requests, "warmup_requests": args.warmup,
               "gpus_measured": len(devices), "devices": devices,
               "sweep_wall_s_measured": round(wall, 3), "worker_prewarm_s": round(prewarm_s, 3),
               "controller_run_s": round(run_s, 3), "convert_s": round(convert_s, 3),
               "sharded_cells": {f"{a}:{b}": k for (a, b), k in shards.items()},
               "cells_started_per_device": per_dev,
               "failed_cells": {j.id: j.failed_cells for j in jobs if j.failed_cells},
               "errors": sweep.errors[:20],
               "jobs_state": {j.id: store.load(j.id).state for j in jobs},
               "actions": [[round(t, 4), a["kind"], a["device"], a["cell"]]
                           for t, a in sweep.actions],
               "cells": cells}
    out.with_suffix(".json").write_text(json.dumps(summary, indent=1))
    print(json.dumps({k: summary[k] for k in ("sweep_wall_s_measured", "worker_prewarm_s",
                                               "controller_run_s", "gpus_measured",
                                               "jobs_state", "errors")}))
    return 0 if all(v == "completed" for v in summary["jobs_state"].values()) else 1


if __name__ == "__main__":
    sys.exit(main())
