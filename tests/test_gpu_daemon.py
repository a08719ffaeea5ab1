"""The controller-driven sweep on a real GPU: real b200
workers, NVML snapshots, self-load exclusion from NVML's process list,
JobStore persistence, and pause/resume when a foreign process loads the GPU
(reference controller.py:150-156, 172-193; profiler/sweep.py:212-216)."""
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import pytest

from paper_2006_05096_b200 import converter, toyformat, zoo
from paper_2006_05096_b200.controller import ControllerConfig
from paper_2006_05096_b200.dispatcher import Dispatcher, b200_template
from paper_2006_05096_b200.hub import Hub, TensorSpec
from paper_2006_05096_b200.profiler.sweep import JobStore, Profiler
from paper_2006_05096_b200.profiler.types import ProfilingJob, SweepSpec
from paper_2006_05096_b200.sweeprun import CellRunner, ControllerSweep, nvml_hooks
from paper_2006_05096_b200.telemetry import NvmlProvider, Telemetry

pytestmark = pytest.mark.gpu

LOAD = r"""
import sys, time, torch
a = torch.randn(8192, 8192, device='cuda', dtype=torch.bfloat16)
for _ in range(3):
    a @ a
torch.cuda.synchronize()
print('go', flush=True)
t0 = time.time()
while time.time() - t0 < float(sys.argv[1]):
    for _ in range(8):
        a @ a
    torch.cuda.synchronize()
print('done', flush=True)
"""


def _register(hub, name):
    if name == "mlp":
        rec = hub.register("mlp", "toy", toyformat.canonical_json(zoo.make_mlp_graph(0)),
                           [TensorSpec("x", [-1, 784])])
        src = "toy"
    else:
        rec = hub.register(name, "torchvision",
                           converter.pack_torchvision(zoo.make_torch_model(name, 0), name),
                           [TensorSpec("x", [-1, 3, 224, 224])])
        src = "torchvision"
    plugin = [p for p in converter.b200_plugins((src,)) if p.target_format == "b200-bf16"][0]
    return rec, hub.convert(rec, plugin)


def _setup(models, batches, n):
    hub = Hub()
    prov = NvmlProvider()
    tel = Telemetry(prov)
    tel.sample_devices()
    disp = Dispatcher(hub, {"b200": b200_template()}, Path(tempfile.mkdtemp()), tel.device_ids)
    tel.instance_pid_resolver = disp.pid_of
    tel.instance_device_resolver = disp.device_of
    store = JobStore(hub.store)
    prof = Profiler(hub, disp, tel, store)
    jobs = []
    for m in models:
        rec, var = _register(hub, m)
        jobs.append(ProfilingJob(f"j-{m}", rec.id, var.id,
                                 SweepSpec(batch_sizes=batches, devices=["gpu:*"],
                                           backends=["b200"], protocols=["grpc-style"],
                                           requests_per_cell=n, warmup_requests=3)))
    for j in jobs:
        store.save(j)
    runner = CellRunner(prof)
    sample, ours_only = nvml_hooks(prov, runner, disp.pid_of)
    return hub, disp, store, runner, jobs, sample, ours_only


def test_controller_sweep_on_gpu0_with_real_workers(gpu_required):
    hub, disp, store, runner, jobs, sample, ours_only = _setup(["mlp", "resnet50"],
                                                               [1, 8, 64], 20)
    sweep = ControllerSweep(["gpu:0"], runner, sample=sample, ours_only=ours_only, quiet_s=0.25,
                            cost_fn=lambda j, c: c.batch_size, jobs_store=store,
                            poll_s=0.005, sample_interval_s=0.02)
    try:
        wall = sweep.run(jobs, timeout_s=300)
    finally:
        runner.shutdown()
        disp.shutdown()
    assert not sweep.errors, sweep.errors
    for j in jobs:
        saved = store.load(j.id)
        assert saved.state == "completed" and len(saved.results) == 3
        assert all(r.device == "gpu:0" and r.peak_throughput > 0 for r in saved.results)
        # the resource columns come from inside the cell (device-timed trace)
        assert all(r.utilization is not None and not r.degraded for r in saved.results)
    # our own workers' NVML load never paused or held back the sweep
    assert not [a for _, a in sweep.actions if a["kind"] == "pause_job"]
    assert not sweep.quiet_samples            # exclusive device: no quiet gaps taken
    assert wall < 60


def test_foreign_load_pauses_then_resumes(gpu_required):
    hub, disp, store, runner, jobs, sample, ours_only = _setup(
        ["resnet50"], [1, 2, 4, 8, 16, 32, 64, 128, 256], 40)
    load = {}
    units = []

    def run_cell(job, unit, dev):
        res = runner(job, unit, dev)
        units.append((time.monotonic(), unit.batch_size))
        if len(units) == 2 and "proc" not in load:
            # a foreign process starts loading the GPU (an online service)
            p = subprocess.Popen([sys.executable, "-c", LOAD, "3.0"], stdout=subprocess.PIPE,
                                 text=True)
            assert p.stdout.readline().strip() == "go"
            load["proc"], load["t_go"] = p, time.monotonic()

            def watch():
                if p.stdout.readline().strip() == "done":   # its last kernel finished
                    load["t_end"] = time.monotonic()
            threading.Thread(target=watch, daemon=True).start()
        return res

    sweep = ControllerSweep(["gpu:0"], run_cell, sample=sample, ours_only=ours_only,
                            quiet_s=0.25, cost_fn=lambda j, c: -c.batch_size, jobs_store=store,
                            poll_s=0.005, sample_interval_s=0.02,
                            config=ControllerConfig(max_cells_per_job=None, order="lpt",
                                                    consecutive_samples=1))
    t0 = time.monotonic()
    try:
        sweep.run(jobs, timeout_s=300)
    finally:
        runner.shutdown()
        disp.shutdown()
        if "proc" in load:
            load["proc"].wait(timeout=60)
    kinds = [a["kind"] for _, a in sweep.actions]
    assert "pause_job" in kinds, (kinds, sweep.quiet_samples)
    assert "resume_job" in kinds[kinds.index("pause_job"):]
    t_pause = t0 + next(t for t, a in sweep.actions if a["kind"] == "pause_job")
    t_resume = t0 + next(t for t, a in sweep.actions if a["kind"] == "resume_job")
    # paused while the load ran, resumed only after its last kernel (the
    # process may still be tearing down its context: idle, so not load)
    assert load["t_go"] <= t_pause <= load["t_end"] <= t_resume + 0.05
    # no cell of ours started on the GPU while the foreign load ran
    starts = [t0 + t for t, a in sweep.actions if a["kind"] == "start_cell"]
    assert not [s for s in starts if t_pause < s < load["t_end"]]
    saved = store.load(jobs[0].id)
    assert saved.state == "completed" and len(saved.results) == 9 and not sweep.errors
