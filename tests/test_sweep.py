"""Profiler.run_sweep control flow (reference sweep.py:196-228): deterministic
order, instance reuse across batch sizes, pause/resume at cell boundaries
(SPEC acceptance 5), failures recorded and skipped, pool cells, CSV schema."""
import csv
import io

import pytest

from paper_2006_05096_b200.dispatcher import ServiceInstance
from paper_2006_05096_b200.errors import CellFailure, RequestFailure
from paper_2006_05096_b200.hub import Hub, ModelVariant, TensorSpec
from paper_2006_05096_b200.profiler import CSV_COLUMNS, results_to_csv
from paper_2006_05096_b200.profiler.stats import LatencySamples
from paper_2006_05096_b200.profiler.sweep import JobStore, Profiler
from paper_2006_05096_b200.profiler.types import ProfilingJob, SweepSpec
from paper_2006_05096_b200.telemetry import InstanceStats


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


class FakeProfiler(Profiler):
    fail_batches = set()

    def measure(self, job, cell, inst, sample_size):
        if cell.batch_size in self.fail_batches:
            raise RequestFailure("boom")
        n = job.sweep.requests_per_cell
        lat = [1.0 + 0.01 * cell.batch_size] * n
        return LatencySamples(lat, [1.1 * (i + 1) for i in range(n)])


def make(devices=("gpu:0",), batches=(1, 2, 4, 8, 16, 32)):
    hub = Hub()
    rec = hub.register("m", "toy", b"weights", [TensorSpec("x", [-1, 784])])
    v = ModelVariant("v1", rec.id, "b200-bf16", hub.put_blob(b"plan"), ["b200"])
    hub.append_variant(rec.id, v)
    hub.advance_status(rec.id, "converting")
    hub.advance_status(rec.id, "converted")
    d = FakeDispatcher()
    jobs = JobStore(hub.store)
    prof = FakeProfiler(hub, d, FakeTelemetry(), jobs)
    job = ProfilingJob("j1", rec.id, "v1", SweepSpec(batch_sizes=list(batches),
                                                    devices=list(devices), backends=["b200"],
                                                    protocols=["grpc-style"],
                                                    requests_per_cell=10, warmup_requests=0))
    return hub, d, jobs, prof, job


def test_full_sweep_and_csv_schema():
    hub, d, jobs, prof, job = make()
    res = prof.run_sweep(job)
    assert [r.batch_size for r in res] == [1, 2, 4, 8, 16, 32]
    assert len(d.dispatched) == 1                       # instance reused across batch sizes
    assert job.state == "completed" and hub.get(job.record_id).status == "profiled"
    rows = list(csv.reader(io.StringIO(results_to_csv(res))))
    assert rows[0] == CSV_COLUMNS and len(rows) == 7
    assert all(r[CSV_COLUMNS.index("resource_scope")] == "gpu:0" for r in rows[1:])


def test_pause_and_resume_exact_remaining_cells():
    hub, d, jobs, prof, job = make()
    calls = []

    def gate(j, cell):
        calls.append(cell.batch_size)
        return len(calls) <= 2
    first = prof.run_sweep(job, should_continue=gate)
    assert len(first) == 2 and job.state == "paused"
    reloaded = jobs.load(job.id)
    second = prof.run_sweep(reloaded)
    assert len(second) == 4                              # exactly the remaining cells
    assert len({r.batch_size for r in reloaded.results}) == 6


def test_failed_cell_recorded_not_retried():
    hub, d, jobs, prof, job = make()
    prof.fail_batches = {4}
    res = prof.run_sweep(job)
    assert len(res) == 5 and list(job.failed_cells) == ["gpu:0|b200|grpc-style|4"]
    assert job.state == "completed"


def test_pool_cells_run_on_resolved_device():
    hub, d, jobs, prof, job = make(devices=("gpu:*",), batches=(1, 2))
    res = prof.run_sweep(job, pool_device=lambda cell: "gpu:3")
    assert {r.device for r in res} == {"gpu:3"}
    assert job.completed_cells == {"gpu:*|b200|grpc-style|1", "gpu:*|b200|grpc-style|2"}


def test_sweep_spec_validation_and_order():
    spec = SweepSpec(batch_sizes=[4, 1], devices=["gpu:1", "gpu:0"], backends=["b200"],
                     protocols=["rest", "grpc-style"])
    keys = [c.key() for c in spec.cells()]
    assert keys[0] == "gpu:0|b200|grpc-style|1" and len(keys) == 8
    from paper_2006_05096_b200.errors import InvalidRequest
    with pytest.raises(InvalidRequest):
        SweepSpec(devices=["gpu:0"], backends=["b200"], requests_per_cell=5).validate()
