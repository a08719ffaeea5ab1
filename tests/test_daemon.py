"""The controller -> profiler daemon glue (sweeprun.ControllerSweep +
CellRunner) on CPU: pause/resume on external load at cell boundaries
(reference controller.py:150-156, 172-193; profiler/sweep.py:212-216),
self-load exclusion, JobStore persistence and resume after a restart,
request-sharded cells, and placement actions."""
import time

import pytest

from paper_2006_05096_b200.controller import ControllerConfig, PlacementRequest
from paper_2006_05096_b200.dispatcher import ServiceInstance
from paper_2006_05096_b200.hub import Hub, ModelVariant, TensorSpec
from paper_2006_05096_b200.profiler.stats import LatencySamples, ShardedSamples, aggregate
from paper_2006_05096_b200.profiler.sweep import JobStore, Profiler
from paper_2006_05096_b200.profiler.types import Cell, ProfilingJob, ProfilingResult, SweepSpec
from paper_2006_05096_b200.sweeprun import (BusyLedger, CellRunner, ControllerSweep,
                                            plan_shards)
from paper_2006_05096_b200.telemetry import InstanceStats, SyntheticProvider

BATCHES = [1, 2, 4, 8, 16, 32, 64, 128, 256]


def pool_job(jid="j", batches=BATCHES, n=10, devices=("gpu:*",)):
    return ProfilingJob(jid, "r" + jid, "v" + jid,
                        SweepSpec(batch_sizes=list(batches), devices=list(devices),
                                  backends=["b200"], protocols=["grpc-style"],
                                  requests_per_cell=n, warmup_requests=0))


def fake_result(job, cell, dev):
    return ProfilingResult(job.variant_id, dev, cell.backend, cell.protocol, cell.batch_size,
                           1.0, 1.0, 1.0, 1.0, None, None)


def util_of(provider):
    return lambda: {d: s.utilization for d, s in provider.sample().items()}


# -- pause / resume on external load -------------------------------------------------

def test_external_load_pauses_at_cell_boundary_and_resumes():
    """gpu:0 is ours; external load appears at 60 ms and leaves at 400 ms.
    The cell running when it appears finishes; its quiet-gap sample sees the
    load -> pause_job; no cell starts while the load lasts; the job resumes
    (resume_job) once the device is idle again and completes."""
    prov = SyntheticProvider([(0, "gpu:0", 0.0, 0, 1), (60, "gpu:0", 0.9, 0, 1),
                              (400, "gpu:0", 0.05, 0, 1)])
    starts = []

    def run_cell(job, cell, dev):
        starts.append(prov.elapsed_ms())
        time.sleep(0.03)
        return fake_result(job, cell, dev)

    states = []
    sweep = ControllerSweep(["gpu:0"], run_cell, sample=util_of(prov),
                            cost_fn=lambda j, c: c.batch_size,
                            on_event=lambda k, p: states.append(p.get("action") or p["state"]))
    job = pool_job()
    sweep.run([job], timeout_s=30)
    kinds = [a["kind"] for _, a in sweep.actions]
    assert "pause_job" in kinds and "resume_job" in kinds
    assert kinds.index("pause_job") < kinds.index("resume_job")
    t_pause = next(t for t, a in sweep.actions if a["kind"] == "pause_job") * 1e3
    t_resume = next(t for t, a in sweep.actions if a["kind"] == "resume_job") * 1e3
    assert t_pause < 200 and t_resume >= 395
    # nothing started on the loaded device between the pause and the load ending
    assert not [s for s in starts if t_pause + 1 < s < 395]
    assert job.is_done() and job.state == "completed" and len(job.results) == 9
    assert "pause_job" in states and "resume_job" in states


def test_exclusive_device_ignores_its_own_nvml_load():
    """All compute processes on the GPU are ours: NVML's 100% is our own
    cell, so the device is re-granted immediately and never paused."""
    sweep = ControllerSweep(["gpu:0"], lambda j, c, d: fake_result(j, c, d),
                            sample=lambda: {"gpu:0": 1.0}, ours_only=lambda d: True,
                            quiet_s=5.0, cost_fn=lambda j, c: c.batch_size)
    job = pool_job()
    t = sweep.run([job], timeout_s=10)
    assert job.is_done() and len(job.results) == 9 and t < 2.0   # no quiet gaps taken
    assert not [a for _, a in sweep.actions if a["kind"] == "pause_job"]


def test_foreign_device_busy_is_never_granted_and_missing_device_is_not_idle():
    used = set()

    def run_cell(job, cell, dev):
        used.add(dev)
        return fake_result(job, cell, dev)

    sweep = ControllerSweep(["gpu:0", "gpu:1", "gpu:2"], run_cell,
                            sample=lambda: {"gpu:0": 0.95, "gpu:1": 0.0},
                            ours_only=lambda d: d != "gpu:0", cost_fn=lambda j, c: c.batch_size)
    job = pool_job()
    sweep.run([job], timeout_s=10)
    assert used == {"gpu:1"} and job.is_done()


def test_busy_ledger_share():
    now = [0.0]
    led = BusyLedger(clock=lambda: now[0])
    led.begin("gpu:0")
    now[0] = 0.1
    led.end("gpu:0")
    now[0] = 0.15
    assert led.share("gpu:0", 0.2) == pytest.approx(0.1 / 0.2)
    now[0] = 0.5
    assert led.share("gpu:0", 0.2) == 0.0


# -- persistence and restart --------------------------------------------------------------

def test_restart_resumes_exact_remaining_cells_from_jobstore():
    hub = Hub()
    store = JobStore(hub.store)
    job = pool_job("jr")
    store.save(job)
    ran = []
    stop_after = 4

    def crashing(job_, cell, dev):
        if len(ran) >= stop_after:
            time.sleep(60)          # the "crash": this cell never finishes
        ran.append(cell.batch_size)
        return fake_result(job_, cell, dev)

    s1 = ControllerSweep(["gpu:0"], crashing, jobs_store=store,
                         cost_fn=lambda j, c: c.batch_size)
    with pytest.raises(TimeoutError):
        s1.run([job], timeout_s=0.5)
    reloaded = store.load("jr")                    # a new daemon process reads the store
    assert len(reloaded.completed_cells) == stop_after and len(reloaded.results) == stop_after
    ran2 = []

    def ok(job_, cell, dev):
        ran2.append(cell.batch_size)
        return fake_result(job_, cell, dev)

    s2 = ControllerSweep(["gpu:0"], ok, jobs_store=store, cost_fn=lambda j, c: c.batch_size)
    s2.run([reloaded], timeout_s=10)
    assert sorted(ran + ran2) == sorted(BATCHES) and not set(ran) & set(ran2)
    final = store.load("jr")
    assert final.state == "completed" and len(final.results) == 9


# -- request shards through the real Profiler ------------------------------------------------

class FakeDispatcher:
    def __init__(self):
        self.dispatched = []
        self.terminated = []

    def dispatch(self, variant, device, backend, protocol):
        inst = ServiceInstance(f"i{len(self.dispatched)}", variant.parent_id, variant.id, device,
                               backend, protocol, endpoint="127.0.0.1:1", state="ready")
        self.dispatched.append(inst)
        return inst

    def terminate(self, iid):
        self.terminated.append(iid)


class FakeTelemetry:
    def sample_instance(self, iid):
        return InstanceStats(iid, 0.0, 0.5, 1 << 30)


class ShardProfiler(Profiler):
    """measure() returns n requests of 2 ms each (+0.5 ms per shard index so
    the per-shard peaks differ), with a device trace like the b200 worker."""
    fail_shard = None

    def measure(self, job, cell, inst, sample_size):
        if self.fail_shard is not None and (cell.batch_size, cell.shard) == self.fail_shard:
            from paper_2006_05096_b200.errors import RequestFailure
            raise RequestFailure("boom")
        n = cell.shard_requests(job.sweep.requests_per_cell)
        lat = 2.0 + 0.5 * cell.shard
        from paper_2006_05096_b200.profiler.stats import ResourceSample
        return LatencySamples([lat] * n, [lat * (i + 1) for i in range(n)], 0,
                              [ResourceSample(lat * i, 0.9, 1 << 30) for i in range(n)])


def make_profiler():
    hub = Hub()
    rec = hub.register("m", "toy", b"weights", [TensorSpec("x", [-1, 784])])
    v = ModelVariant("v1", rec.id, "b200-bf16", hub.put_blob(b"plan"), ["b200"])
    hub.append_variant(rec.id, v)
    hub.advance_status(rec.id, "converting")
    hub.advance_status(rec.id, "converted")
    store = JobStore(hub.store)
    disp = FakeDispatcher()
    return hub, store, disp, ShardProfiler(hub, disp, FakeTelemetry(), store)


def test_plan_shards_splits_only_makespan_bounding_cells():
    jobs = [pool_job("a", n=100), pool_job("b", batches=[1, 2], n=100)]
    cost = lambda j, c: c.batch_size * (100.0 if j.id == "a" else 1.0)
    plan = plan_shards(jobs, 8, cost)
    # total 51103; bound = 0.5 * total / 8 = 3194: a@32 (3200) and up are split
    assert plan == {("a", "gpu:*|b200|grpc-style|256"): 8,
                    ("a", "gpu:*|b200|grpc-style|128"): 5,
                    ("a", "gpu:*|b200|grpc-style|64"): 3,
                    ("a", "gpu:*|b200|grpc-style|32"): 2}
    units = jobs[0].remaining_units()
    assert len(units) == 5 + 2 + 3 + 5 + 8
    assert Cell.from_key("gpu:*|b200|grpc-style|256#3/8") == \
        Cell("gpu:*", "b200", "grpc-style", 256, 3, 8)
    assert sum(Cell("gpu:*", "b", "p", 1, i, 8).shard_requests(100) for i in range(8)) == 100
    assert plan_shards([pool_job("c")], 1, cost) == {}


def test_sharded_cells_merge_through_controller_sweep():
    hub, store, disp, prof = make_profiler()
    job = ProfilingJob("js", hub._records and next(iter(hub._records)), "v1",
                       SweepSpec(batch_sizes=[64, 256], devices=["gpu:*"], backends=["b200"],
                                 protocols=["grpc-style"], requests_per_cell=100,
                                 warmup_requests=0))
    job.shard_plan = {"gpu:*|b200|grpc-style|256": 4}
    store.save(job)
    runner = CellRunner(prof)
    devices = [f"gpu:{i}" for i in range(4)]
    sweep = ControllerSweep(devices, runner, jobs_store=store,
                            cost_fn=lambda j, c: c.batch_size / c.shards)
    sweep.run([job], timeout_s=20)
    runner.shutdown()
    assert job.is_done() and not job.shard_samples and not sweep.errors
    r256 = next(r for r in job.results if r.batch_size == 256)
    assert r256.raw_sample_count == 100                      # union of the 4 shards
    # peak = max of per-shard peaks (shard 0: 2.0 ms/request), not the pooled rate
    assert r256.peak_throughput == pytest.approx(256 * 1000 / 2.0, rel=1e-9)
    assert set(r256.device.split(",")) <= set(devices) and len(r256.device.split(",")) >= 2
    assert r256.p99_latency_ms == pytest.approx(3.5)
    # an instance per (variant, device) is reused across cells (model affinity)
    assert len(disp.dispatched) == len({i.device for i in disp.dispatched})
    assert store.load("js").state == "completed"
    # the shards' placements were distinct units granted concurrently
    shard_keys = [k for k, _ in sweep.placements if "#" in k]
    assert sorted(shard_keys) == [f"gpu:*|b200|grpc-style|256#{i}/4" for i in range(4)]


def test_sharded_samples_peak_is_max_of_shard_peaks():
    a = LatencySamples([1.0] * 10, [1.0 * (i + 1) for i in range(10)])
    b = LatencySamples([2.0] * 10, [2.0 * (i + 1) for i in range(10)])
    r = aggregate(ShardedSamples([a, b]), [], 8, variant_id="v", device="gpu:0,gpu:1",
                  backend="b200", protocol="grpc-style")
    assert r.raw_sample_count == 20 and r.peak_throughput == pytest.approx(8000.0)
    assert r.p50_latency_ms == 1.0 and r.p99_latency_ms == 2.0


def test_failed_shard_fails_its_cell_once_and_sweep_goes_on():
    hub, store, disp, prof = make_profiler()
    prof.fail_shard = (256, 1)
    rid = next(iter(hub._records))
    job = ProfilingJob("jf", rid, "v1",
                       SweepSpec(batch_sizes=[64, 256], devices=["gpu:*"], backends=["b200"],
                                 protocols=["grpc-style"], requests_per_cell=40,
                                 warmup_requests=0))
    job.shard_plan = {"gpu:*|b200|grpc-style|256": 2}
    prof.run_sweep(job, pool_device=lambda c: "gpu:0")
    assert list(job.failed_cells) == ["gpu:*|b200|grpc-style|256"]
    assert [r.batch_size for r in job.results] == [64] and not job.shard_samples
    assert job.state == "completed"


def test_shard_progress_survives_restart():
    hub, store, disp, prof = make_profiler()
    rid = next(iter(hub._records))
    job = ProfilingJob("jp", rid, "v1",
                       SweepSpec(batch_sizes=[256], devices=["gpu:*"], backends=["b200"],
                                 protocols=["grpc-style"], requests_per_cell=30,
                                 warmup_requests=0))
    job.shard_plan = {"gpu:*|b200|grpc-style|256": 3}
    calls = []
    prof.run_sweep(job, should_continue=lambda j, c: len(calls) < 2 and not calls.append(c),
                   pool_device=lambda c: "gpu:0")
    saved = store.load("jp")
    assert saved.state == "paused" and len(saved.shard_samples) == 2
    assert [u.key() for u in saved.remaining_units()] == ["gpu:*|b200|grpc-style|256#2/3"]
    prof.run_sweep(saved, pool_device=lambda c: "gpu:1")
    assert saved.state == "completed" and saved.results[0].raw_sample_count == 30
    assert saved.results[0].device == "gpu:0,gpu:1"


# -- placements ------------------------------------------------------------------------------

def test_place_instance_goes_to_least_utilised_idle_device():
    placed = []
    sweep = ControllerSweep(["gpu:0", "gpu:1"], lambda j, c, d: fake_result(j, c, d),
                            sample=lambda: {"gpu:0": 0.3, "gpu:1": 0.1},
                            on_place=lambda pid, rid, dev: placed.append((pid, dev)),
                            config=ControllerConfig(max_cells_per_job=None, order="lpt",
                                                    consecutive_samples=1, idle_threshold=0.4))
    sweep.ctrl.request_placement(PlacementRequest("p1", "rec", "var", "b200", "grpc-style"))
    sweep.run([pool_job(batches=[1])], timeout_s=5)
    assert placed and placed[0][0] == "p1" and placed[0][1] in ("gpu:0", "gpu:1")
