"""Controller: the SPEC examples, the acceptance-4 safety
property over randomized traces, the reference NameError path, and the
multi-GPU extensions (per-device concurrency, pool cells, LPT)."""
import random

import pytest

from paper_2006_05096_b200.controller import (Controller, ControllerConfig, PlacementRequest)
from paper_2006_05096_b200.errors import InvalidRequest
from paper_2006_05096_b200.profiler.types import ProfilingJob, SweepSpec
from paper_2006_05096_b200.telemetry import DeviceSnapshot, DeviceStats


def snap(utils, stale=False):
    return DeviceSnapshot(0.0, {d: DeviceStats(u, 0, 1) for d, u in utils.items()}, stale)


def job(jid, devices, batches=(1, 2), backend="b200"):
    return ProfilingJob(id=jid, record_id="r" + jid, variant_id="v" + jid,
                        sweep=SweepSpec(batch_sizes=list(batches), devices=list(devices),
                                        backends=[backend], protocols=["grpc-style"]))


def feed(c, utils, n=3):
    for _ in range(n):
        c.on_snapshot(snap(utils))


def test_idle_examples():
    c = Controller()
    feed(c, {"gpu:0": 0.3})
    assert c.is_idle("gpu:0")
    c2 = Controller()
    feed(c2, {"gpu:0": 0.45})
    assert not c2.is_idle("gpu:0")
    for trace, idle in (([0.35, 0.42, 0.39], False), ([0.35, 0.38, 0.39], True)):
        c3 = Controller()
        for u in trace:
            c3.on_snapshot(snap({"gpu:0": u}))
        assert c3.is_idle("gpu:0") == idle


def test_ring_keeps_k_and_staleness():
    c = Controller()
    feed(c, {"gpu:0": 0.0, "gpu:1": 0.0})
    for _ in range(3):
        c.on_snapshot(snap({"gpu:0": 0.0}))     # gpu:1 absent -> goes stale
    assert c.is_idle("gpu:0") and not c.is_idle("gpu:1")
    assert len(c._windows["gpu:0"]) == 3
    c.on_snapshot(snap({}, stale=True))
    assert c._seq == 7


def test_tick_examples():
    c = Controller()
    feed(c, {"gpu:0": 0.0})
    assert c.tick() == []                       # no jobs
    c = Controller()
    feed(c, {"cpu:0": 0.45})
    j = job("a", ["cpu:0"])
    c.submit(j)
    assert c.tick() == [] and j.state == "waiting_for_device"
    c = Controller()
    feed(c, {"gpu:0": 0.0, "gpu:1": 0.0})
    a, b = job("a", ["gpu:0", "gpu:1"]), job("b", ["gpu:0", "gpu:1"])
    c.submit(a)
    c.submit(b)
    acts = [x for x in c.tick() if x.kind == "start_cell"]
    assert [(x.device, x.job_id) for x in acts] == [("gpu:0", "a"), ("gpu:1", "b")]


def test_placement_no_longer_raises_nameerror():
    # reference controller.py:232 raised NameError here
    c = Controller()
    feed(c, {"gpu:0": 0.1, "gpu:1": 0.05})
    c.request_placement(PlacementRequest("p1", "r", "v", "b200", "grpc-style"))
    acts = c.tick()
    assert [(x.kind, x.device) for x in acts] == [("place_instance", "gpu:1")]


def test_placement_skips_devices_granted_this_tick():
    c = Controller()
    feed(c, {"gpu:0": 0.0, "gpu:1": 0.1})
    c.submit(job("a", ["gpu:0"]))
    c.request_placement(PlacementRequest("p1", "r", "v", "b200", "grpc-style"))
    acts = c.tick()
    assert ("start_cell", "gpu:0") in [(x.kind, x.device) for x in acts]
    assert [x.device for x in acts if x.kind == "place_instance"] == ["gpu:1"]


def test_pause_with_self_load_exclusion():
    c = Controller()
    feed(c, {"gpu:0": 0.0})
    j = job("a", ["gpu:0"])
    c.submit(j)
    c.tick()
    c.note_instance_stats("gpu:0", 0.9)         # our own load
    feed(c, {"gpu:0": 0.95})
    assert not any(x.kind == "pause_job" for x in c.tick())
    c.note_instance_stats("gpu:0", 0.1)
    assert [x.kind for x in c.tick()] == ["pause_job"] and j.state == "paused"


def test_safety_over_randomized_traces():
    """Acceptance criterion 4: no start_cell on a non-idle device; a job whose
    device stays above tau for K samples is paused within one tick."""
    rng = random.Random(1234)
    for _ in range(300):
        c = Controller(ControllerConfig(max_cells_per_job=rng.choice([1, None])))
        devs = [f"gpu:{i}" for i in range(rng.randint(1, 4))]
        jobs = [job(str(i), rng.sample(devs, rng.randint(1, len(devs))), (1, 2, 4))
                for i in range(rng.randint(1, 4))]
        for j in jobs:
            c.submit(j)
        hot = {d: 0 for d in devs}
        for _ in range(rng.randint(5, 25)):
            u = {d: rng.choice([0.1, 0.2, 0.5, 0.9]) for d in devs if rng.random() < 0.95}
            c.on_snapshot(snap(u))
            for d in devs:
                hot[d] = hot[d] + 1 if u.get(d, 0) > 0.4 else 0
            idle_before = {d: c.is_idle(d) for d in devs}
            running_before = {d: (jid, c.job(jid).state)
                              for d, (jid, _) in c.running_cells().items()}
            acts = c.tick()
            for a in acts:
                if a.kind == "start_cell":
                    assert idle_before[a.device]
            paused = {(a.device, a.job_id) for a in acts if a.kind == "pause_job"}
            for d, (jid, state) in running_before.items():
                if hot[d] >= 3 and state == "running" and (d, jid) not in paused:
                    pytest.fail("busy device did not pause its job")
            for d in list(c.running_cells()):
                if rng.random() < 0.5:
                    jid, cell = c.running_cells()[d]
                    c.job(jid).completed_cells.add(cell.key())
                    c.note_cell_done(d)


def test_reference_mode_one_cell_per_job_caps_devices():
    c = Controller()
    feed(c, {f"gpu:{i}": 0.0 for i in range(8)})
    for i in range(5):
        c.submit(job(str(i), [f"gpu:{d}" for d in range(8)]))
    starts = [a for a in c.tick() if a.kind == "start_cell"]
    assert len(starts) == 5                      # 5 jobs -> 5 GPUs


def test_pool_cells_fill_all_devices():
    c = Controller(ControllerConfig(max_cells_per_job=None, order="lpt"),
                   cost_fn=lambda j, cell: cell.batch_size)
    feed(c, {f"gpu:{i}": 0.0 for i in range(8)})
    j = job("a", ["gpu:*"], batches=(1, 2, 4, 8, 16, 32, 64, 128, 256))
    c.submit(j)
    starts = [a for a in c.tick() if a.kind == "start_cell"]
    assert len(starts) == 8
    assert [s.cell.batch_size for s in starts] == [256, 128, 64, 32, 16, 8, 4, 2]   # LPT
    assert len({s.cell.key() for s in starts}) == 8          # no pool cell granted twice


def test_config_validation():
    with pytest.raises(InvalidRequest):
        Controller(ControllerConfig(idle_threshold=0))
    with pytest.raises(InvalidRequest):
        Controller(ControllerConfig(order="random"))
