"""C5 elastic evaluation on this box (BASELINE configs[4]): a ResNet-50 bf16
online-serving load holds a p99 SLO while profiling jobs arrive.

The serving load (``--load device``, default) is GPU-bound: back-to-back
requests of ``--serve-batch`` images inside the serving worker, each copying
its inputs host->device from pinned memory and its outputs back, timed on
the device (online.device_loop_load) — request latency includes any time the
GPU gives another process.  ``--load binary`` drives closed-loop binary
predict clients over TCP instead (online.closed_loop_load); on one host that
load is bound by Python socket copies of 0.6 MB/image and keeps the GPU ~8%
busy, so it cannot show interference.

Three phases on gpu:0, serving load running throughout phases 1-3:
  1. serving alone                          -> the p99 baseline, SLO = slo_x * that
  2. profiling co-located WITHOUT gating    -> what an SLO-blind scheduler does
     (ControllerSweep told every GPU is idle)
  3. profiling under the idle-aware controller (NVML snapshots, self-load
     exclusion): the serving worker is a foreign process keeping the GPU
     busy, so no profiling cell is granted there while it serves; the load
     then stops and the queued profiling completes on the now idle GPU.
Writes <out>.json: per-window serving p50/p99 and SLO verdicts, NVML
utilisation while serving, the controller's actions and the profiling
completion times.

    python tools/elastic_c5.py gpurun_out/r2_c5
"""
import argparse
import json
import os
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.pop("B2_DEV", None)

import numpy as np  # noqa: E402

from paper_2006_05096_b200 import converter, zoo  # noqa: E402
from paper_2006_05096_b200.controller import ControllerConfig  # noqa: E402
from paper_2006_05096_b200.dispatcher import Dispatcher, b200_template  # noqa: E402
from paper_2006_05096_b200.hub import Hub, TensorSpec  # noqa: E402
from paper_2006_05096_b200.online import (closed_loop_load, device_loop_load,  # noqa: E402
                                          slo_report)
from paper_2006_05096_b200.profiler.sweep import JobStore, Profiler  # noqa: E402
from paper_2006_05096_b200.profiler.types import ProfilingJob, SweepSpec  # noqa: E402
from paper_2006_05096_b200.sweeprun import CellRunner, ControllerSweep, nvml_hooks  # noqa: E402
from paper_2006_05096_b200.telemetry import NvmlProvider, Telemetry  # noqa: E402


def register(hub, name):
    rec = hub.register(name, "torchvision",
                       converter.pack_torchvision(zoo.make_torch_model(name, 0), name),
                       [TensorSpec("x", [-1, 3, 224, 224])])
    plugin = [p for p in converter.b200_plugins(("torchvision",))
              if p.target_format == "b200-bf16"][0]
    return rec, hub.convert(rec, plugin)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--serve-batch", type=int, default=16)
    ap.add_argument("--clients", type=int, default=8)
    ap.add_argument("--phase-s", type=float, default=4.0)
    ap.add_argument("--slo-x", type=float, default=1.5)
    ap.add_argument("--requests", type=int, default=100)
    ap.add_argument("--load", choices=["device", "binary"], default="device")
    args = ap.parse_args()

    hub = Hub()
    prov = NvmlProvider()
    tel = Telemetry(prov)
    tel.sample_devices()
    extra = ("--max-batch", "128", "--batch-timeout-ms", "1.0") if args.load == "binary" else ()
    disp = Dispatcher(hub, {"b200": b200_template(extra_args=extra)},
                      Path(tempfile.mkdtemp()), tel.device_ids)
    tel.instance_pid_resolver = disp.pid_of
    tel.instance_device_resolver = disp.device_of
    store = JobStore(hub.store)
    prof = Profiler(hub, disp, tel, store)
    serve_rec, serve_var = register(hub, "resnet50")
    prof_models = ["resnet50", "vgg16", "mobilenet_v2"]
    variants = {m: register(hub, m) for m in prof_models}

    # the online service: its own worker process on gpu:0 (foreign to the profiler)
    svc = disp.dispatch(serve_var, "gpu:0", "b200", "grpc-style")
    rng = np.random.default_rng(0)
    batches = [rng.standard_normal((args.serve_batch, 3 * 224 * 224), dtype=np.float32)
               for _ in range(args.clients if args.load == "binary" else 0)]
    stop = threading.Event()
    load = {}
    util = []

    def serve_load():
        if args.load == "device":
            load["res"] = device_loop_load(svc.endpoint, args.serve_batch, stop=stop)
        else:
            load["res"] = closed_loop_load(svc.endpoint, lambda i: batches[i],
                                           concurrency=args.clients, stop=stop,
                                           warmup_requests=3)

    def sampler():
        while not stop.is_set():
            util.append((time.monotonic(), prov.sample()["gpu:0"].utilization))
            time.sleep(0.05)

    def jobs(tag):
        out = []
        for m in prof_models:
            rec, var = variants[m]
            j = ProfilingJob(f"{tag}-{m}", rec.id, var.id,
                             SweepSpec(batch_sizes=[1, 16, 64, 256], devices=["gpu:*"],
                                       backends=["b200"], protocols=["grpc-style"],
                                       requests_per_cell=args.requests, warmup_requests=10))
            store.save(j)
            out.append(j)
        return out

    runner = CellRunner(prof)
    sample, ours_only = nvml_hooks(prov, runner, disp.pid_of)
    tl = threading.Thread(target=serve_load, daemon=True)
    ts = threading.Thread(target=sampler, daemon=True)
    tl.start()
    ts.start()
    t_start = time.monotonic()
    time.sleep(args.phase_s)                                  # phase 1: serving alone
    t1 = time.monotonic()

    # phase 2: SLO-blind co-location (every GPU reported idle, no exclusion)
    naive_jobs = jobs("naive")
    naive = ControllerSweep(["gpu:0"], runner, sample=lambda: {"gpu:0": 0.0},
                            ours_only=lambda d: True, cost_fn=lambda j, c: c.batch_size,
                            jobs_store=store)
    naive_s = naive.run(naive_jobs, timeout_s=600)
    t2 = time.monotonic()
    time.sleep(0.5)
    t2b = time.monotonic()

    # phase 3: the idle-aware controller; the load stops after phase_s
    ctrl_jobs = jobs("ctrl")
    ctrl = ControllerSweep(["gpu:0"], runner, sample=sample, ours_only=ours_only, quiet_s=0.25,
                           cost_fn=lambda j, c: c.batch_size, jobs_store=store,
                           poll_s=0.005, sample_interval_s=0.05,
                           config=ControllerConfig(max_cells_per_job=None, order="lpt",
                                                   consecutive_samples=3, idle_threshold=0.4))
    t_stop = {}

    def stop_later():
        time.sleep(args.phase_s)
        t_stop["t"] = time.monotonic()
        stop.set()

    threading.Thread(target=stop_later, daemon=True).start()
    ctrl_s = ctrl.run(ctrl_jobs, timeout_s=600)
    t3 = time.monotonic()
    tl.join(timeout=60)
    runner.shutdown()
    disp.shutdown()

    res = load["res"]
    base_p99 = res.p(99, t_start + 0.5, t1)
    slo = args.slo_x * base_p99
    windows = [("1_serving_alone", t_start + 0.5, t1), ("2_naive_colocation", t1, t2),
               ("3_controller_while_serving", t2b, t_stop["t"])]
    first_ctrl_start = None
    for t, a in ctrl.actions:
        if a["kind"] == "start_cell":
            first_ctrl_start = t2b + t
            break
    u_serv = [u for t, u in util if t_start + 0.5 <= t < t1]
    out = {
        "config": f"C5 elastic: ResNet-50 bf16 serving on gpu:0, b={args.serve_batch}, load "
                  + ("device (back-to-back requests with pinned H2D/D2H, CUDA-event timed)"
                     if args.load == "device" else
                     f"{args.clients} closed-loop binary clients, worker dynamic batching <= 128")
                  + f"; profiling jobs {prof_models} x b in {{1,16,64,256}}, n={args.requests}",
        "slo_ms": round(slo, 3), "slo_rule": f"{args.slo_x} x p99 of serving alone",
        "windows": slo_report(res, slo, windows),
        "nvml_util_serving_alone": {"median": float(np.median(u_serv)) if u_serv else None,
                                    "samples": len(u_serv)},
        "naive": {"profiling_s": round(naive_s, 3),
                  "cells": sum(len(j.results) for j in naive_jobs)},
        "controller": {"run_s": round(ctrl_s, 3),
                       "cells": sum(len(j.results) for j in ctrl_jobs),
                       "first_grant_after_load_stop_s":
                           None if first_ctrl_start is None else
                           round(first_ctrl_start - t_stop["t"], 3),
                       "cells_granted_while_serving":
                           sum(1 for t, a in ctrl.actions if a["kind"] == "start_cell"
                               and t2b + t < t_stop["t"]),
                       "jobs_state": {j.id: store.load(j.id).state for j in ctrl_jobs},
                       "actions": [[round(t, 3), a["kind"], a["cell"]] for t, a in
                                   ctrl.actions][:60]},
    }
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).with_suffix(".json").write_text(json.dumps(out, indent=1))
    print(json.dumps({k: out[k] for k in ("slo_ms", "windows", "nvml_util_serving_alone")}))
    print(json.dumps({k: v for k, v in out["controller"].items() if k != "actions"}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
