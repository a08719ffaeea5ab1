"""Online serving path on CPU: binary
predict frames through the worker's frame server, the closed-loop serving
load and its SLO windows, the dynamic batcher, the fault script
(reference mockserve/server.py:59-88, 183-203; clients.py:76-124)."""
import socket
import struct
import threading
import time

import numpy as np
import pytest

from paper_2006_05096_b200 import wire
from paper_2006_05096_b200.errors import RequestFailure
from paper_2006_05096_b200.online import (BinaryClient, DynamicBatcher, closed_loop_load,
                                          slo_report)
from paper_2006_05096_b200.worker import Executor, FaultScript, serve


class FakePlan:
    in_dtype = np.float32
    in_elems = 4
    out_elems = 2
    in_kind = 0
    dtype = 1
    flops_per_sample = 16
    weight_bytes = 0
    launches_per_forward = 1

    def __init__(self, delay_s=0.0):
        self.delay_s = delay_s
        self.calls = []

    def predict(self, x):
        self.calls.append(x.shape[0])
        time.sleep(self.delay_s)
        return (x[:, :2] * 2.0).astype(np.float32)


class FakeExecutor(Executor):
    def __init__(self, plan, fault=None, max_batch=0, timeout_ms=2.0):
        self.plan = plan
        self.meta = {"model": "fake"}
        self.fault_script = fault or FaultScript([])
        self.started = time.monotonic()
        self.batcher = DynamicBatcher(plan.predict, max_batch, timeout_ms) if max_batch else None


@pytest.fixture
def server():
    made = []

    def start(ex):
        srv = serve(ex, "grpc-style")
        threading.Thread(target=srv.serve_forever, daemon=True).start()
        made.append(srv)
        return f"127.0.0.1:{srv.server_address[1]}"

    yield start
    for s in made:
        s.shutdown()
        s.server_close()


def test_predict_bin_roundtrip(server):
    ep = server(FakeExecutor(FakePlan()))
    cli = BinaryClient.to(ep)
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    y, head = cli.predict(x)
    assert np.array_equal(y, x[:, :2] * 2) and head["batch"] == 3 and head["ok"]
    with pytest.raises(RequestFailure, match="does not match"):
        cli.predict(np.zeros((2, 5), np.float32))       # wrong sample size -> worker error
    cli.close()


def test_closed_loop_load_and_slo_windows(server):
    ep = server(FakeExecutor(FakePlan(delay_s=0.002)))
    res = closed_loop_load(ep, lambda i: np.ones((2, 4), np.float32), concurrency=3,
                           n_requests=60, warmup_requests=1)
    assert len(res.latencies_ms) == 60 and res.failed == 0
    assert all(lat >= 2.0 for lat in res.latencies_ms)
    s = res.samples()
    assert s.completions_ms == sorted(s.completions_ms)
    mid = res.wall_done[0] + (res.wall_done[-1] - res.wall_done[0]) / 2
    rep = slo_report(res, 50.0, [("all", res.t0, None), ("late", mid, None)])
    assert rep["all"]["requests"] == 60 and rep["all"]["slo_held"]
    assert 0 < rep["late"]["requests"] < 60
    assert slo_report(res, 0.5, [("all", res.t0, None)])["all"]["slo_held"] is False


def test_closed_loop_load_stops_on_event(server):
    ep = server(FakeExecutor(FakePlan(delay_s=0.001)))
    stop = threading.Event()
    threading.Timer(0.2, stop.set).start()
    res = closed_loop_load(ep, lambda i: np.ones((1, 4), np.float32), concurrency=2, stop=stop)
    assert len(res.latencies_ms) > 10


def test_load_aborts_when_failures_exceed_budget():
    with pytest.raises(RequestFailure, match="aborted"):
        closed_loop_load("127.0.0.1:1", lambda i: np.ones((1, 4), np.float32),
                         n_requests=20, warmup_requests=0, timeout_s=1.0)


def test_dynamic_batcher_merges_concurrent_requests():
    plan = FakePlan(delay_s=0.01)
    b = DynamicBatcher(plan.predict, max_batch=8, timeout_ms=20.0)
    outs = {}

    def go(i):
        x = np.full((2, 4), float(i), np.float32)
        outs[i] = b.submit(x)

    ts = [threading.Thread(target=go, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    b.close()
    assert sum(plan.calls) == 8 and len(plan.calls) < 4          # merged forwards
    for i, (y, ms, merged) in outs.items():
        assert np.array_equal(y, np.full((2, 2), 2.0 * i)) and merged >= 2
    assert max(plan.calls) <= 8


def test_dynamic_batcher_caps_and_errors():
    def boom(x):
        raise ValueError("kernel failed")
    b = DynamicBatcher(boom, max_batch=4, timeout_ms=1.0)
    with pytest.raises(ValueError, match="kernel failed"):
        b.submit(np.zeros((1, 4), np.float32))
    b.close()
    plan = FakePlan()
    b = DynamicBatcher(plan.predict, max_batch=4, timeout_ms=1.0)
    y, _, merged = b.submit(np.zeros((6, 4), np.float32))   # larger than max: runs alone
    assert y.shape == (6, 2) and merged == 6
    b.close()
    with pytest.raises(ValueError):
        DynamicBatcher(plan.predict, 0)


def test_worker_batcher_through_frames(server):
    plan = FakePlan(delay_s=0.005)
    ep = server(FakeExecutor(plan, max_batch=16, timeout_ms=10.0))
    res = closed_loop_load(ep, lambda i: np.full((2, 4), float(i), np.float32), concurrency=4,
                           n_requests=40, warmup_requests=0)
    assert len(res.latencies_ms) == 40 and max(plan.calls) > 2   # some forwards merged


def test_fault_script_health(server, tmp_path):
    f = tmp_path / "faults"
    f.write_text("# t_ms action\n0 health_ok\n50 health_fail\n150 health_ok\n")
    fs = FaultScript.from_file(f)
    assert fs.healthy_at(10) and not fs.healthy_at(60) and fs.healthy_at(200)
    with pytest.raises(ValueError):
        FaultScript([(0.0, "explode")])
    ep = server(FakeExecutor(FakePlan(), fault=FaultScript([(0.0, "health_fail")])))
    host, port = ep.split(":")
    s = socket.create_connection((host, int(port)))
    wire.write_frame(s, b'{"kind": "health"}')
    import json
    assert json.loads(wire.read_frame(s)) == {"ok": False, "status": "unhealthy"}
    s.close()


def test_oversized_json_frame_rejected_from_header(server):
    """A frame over the JSON limit that does not announce itself as binary is
    refused after reading 4 body bytes, not buffered."""
    ep = server(FakeExecutor(FakePlan()))
    host, port = ep.split(":")
    s = socket.create_connection((host, int(port)))
    s.sendall(struct.pack(">I", wire.MAX_JSON_FRAME + 100) + b'{"ki')
    s.settimeout(5)
    assert s.recv(16) == b""          # the worker dropped the connection
    s.close()


class BenchPlan(FakePlan):
    def bench(self, batch, n, warm, seed, e2e=False):
        lat = np.full(n, 0.5)
        return lat, np.cumsum(lat)

    def device_bytes(self):
        return 1 << 20


def test_device_loop_load_maps_device_completions_to_wall_time(server):
    from paper_2006_05096_b200.online import device_loop_load
    ep = server(FakeExecutor(BenchPlan()))
    res = device_loop_load(ep, 16, requests_per_call=10, n_calls=3)
    assert len(res.latencies_ms) == 30 and all(v == 0.5 for v in res.latencies_ms)
    assert res.wall_done == sorted(res.wall_done) or len(set(res.wall_done)) > 1
    assert res.p(99) == 0.5
    stop = threading.Event()
    stop.set()
    assert len(device_loop_load(ep, 16, stop=stop).latencies_ms) == 0
