"""Online serving path: binary predict client, closed-loop serving load, and
the worker-side dynamic batcher (config C5).

The reference serves JSON lists (mockserve/server.py:117-127 behind the
grpc-style framing server.py:183-203, client clients.py:76-124): a ResNet-50
image batch at b >= 90 overflows its 64 MiB frame and JSON decoding alone
costs seconds.  Here a request is one ``predict_bin`` frame (wire.py): raw
fp32 (or int64 token) samples in, raw fp32 outputs out, over one TCP_NODELAY
connection per client thread.

* ``BinaryClient`` — one connection, ``predict(x) -> (y, header)``.
* ``closed_loop_load`` — the serving load of C5: ``concurrency`` client
  threads, each sending its next request as soon as the previous reply
  arrives, for a fixed request count or until stopped; per-request latency
  and wall-clock completion (so p99 can be read per time window, e.g. while a
  profiling cell shares the GPU).  Same failure budget as the reference's
  ``measure_cell`` (clients.py:161-255).
* ``DynamicBatcher`` — used by the worker (``--max-batch``): concurrent
  requests that arrive within ``timeout_ms`` of the first are concatenated
  into one forward (up to ``max_batch`` samples) and the outputs split back,
  trading a bounded queueing delay for fewer, larger forwards.
"""

from __future__ import annotations

import socket
import threading
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import wire
from .errors import RequestFailure
from .profiler.clients import split_endpoint
from .profiler.stats import LatencySamples, percentile


class BinaryClient:
    """predict_bin frames over one TCP connection."""

    def __init__(self, host: str, port: int, timeout_s: float = 30.0):
        self.host, self.port, self.timeout_s = host, port, timeout_s
        self._sock = socket.create_connection((host, port), timeout=timeout_s)
        wire.nodelay(self._sock)

    @classmethod
    def to(cls, endpoint: str, timeout_s: float = 30.0) -> "BinaryClient":
        host, port = split_endpoint(endpoint)
        return cls(host, port, timeout_s)

    def predict(self, x: np.ndarray) -> tuple[np.ndarray, dict]:
        x = np.ascontiguousarray(x)
        if x.ndim != 2 or x.shape[0] < 1:
            raise ValueError(f"expected a non-empty [batch, elems] array, got {x.shape}")
        dt = "i64" if x.dtype == np.int64 else "f32"
        if dt == "f32" and x.dtype != np.float32:
            x = x.astype(np.float32)
        frame = wire.pack_bin({"kind": "predict_bin", "batch": int(x.shape[0]), "dtype": dt},
                              x.data)
        wire.write_frame(self._sock, frame)
        raw = wire.read_frame(self._sock)
        if raw is None:
            raise RequestFailure("connection closed by the worker")
        if not raw.startswith(wire.BIN_MAGIC):
            import json
            raise RequestFailure(f"worker error: {json.loads(raw).get('error')}")
        head, body = wire.unpack_bin(raw)
        y = np.frombuffer(body, dtype=np.float32).reshape(head["batch"], head["out_elems"])
        return y, head

    def close(self) -> None:
        try:
            self._sock.close()
        except OSError:
            pass


@dataclass
class LoadResult:
    """Per-request record of a serving load (ms; wall = time.monotonic())."""

    latencies_ms: list = field(default_factory=list)
    completions_ms: list = field(default_factory=list)     # since the load's start
    wall_done: list = field(default_factory=list)          # monotonic seconds
    service_ms: list = field(default_factory=list)         # worker-side time per request
    failed: int = 0
    t0: float = 0.0

    def samples(self) -> LatencySamples:
        order = np.argsort(self.completions_ms, kind="stable")
        return LatencySamples([self.latencies_ms[i] for i in order],
                              [self.completions_ms[i] for i in order], self.failed)

    def p(self, q, t_from: Optional[float] = None, t_to: Optional[float] = None) -> float:
        """Nearest-rank percentile (the reference's percentile()) of the
        requests completing in [t_from, t_to) (monotonic seconds)."""
        lat = [lat for lat, w in zip(self.latencies_ms, self.wall_done)
               if (t_from is None or w >= t_from) and (t_to is None or w < t_to)]
        return percentile(lat, q) if lat else float("nan")

    def count(self, t_from: Optional[float] = None, t_to: Optional[float] = None) -> int:
        return sum(1 for w in self.wall_done
                   if (t_from is None or w >= t_from) and (t_to is None or w < t_to))


def closed_loop_load(endpoint: str, make_batch: Callable[[int], np.ndarray], *,
                     concurrency: int = 1, n_requests: Optional[int] = None,
                     stop: Optional[threading.Event] = None, warmup_requests: int = 2,
                     max_failure_fraction: float = 0.05,
                     timeout_s: float = 30.0) -> LoadResult:
    """Closed-loop binary-predict load.  Ends after ``n_requests`` timed
    requests (split over the threads) or when ``stop`` is set."""
    if n_requests is None and stop is None:
        raise ValueError("give n_requests or a stop event")
    res = LoadResult()
    lock = threading.Lock()
    counts = None
    if n_requests is not None:
        counts = [n_requests // concurrency + (i < n_requests % concurrency)
                  for i in range(concurrency)]
    abort = threading.Event()
    budget = [int(max_failure_fraction * n_requests) if n_requests else 1 << 30]
    barrier = threading.Barrier(concurrency,
                                action=lambda: setattr(res, "t0", time.monotonic()))

    def run(idx: int):
        x = make_batch(idx)
        try:
            cli = BinaryClient.to(endpoint, timeout_s)
        except OSError:
            cli = None
        try:
            for _ in range(warmup_requests):
                if cli is not None:
                    try:
                        cli.predict(x)
                    except (OSError, RequestFailure, ValueError):
                        pass
            try:
                barrier.wait(timeout=timeout_s * (warmup_requests + 1))
            except threading.BrokenBarrierError:
                return
            k = 0
            while not abort.is_set():
                if counts is not None and k >= counts[idx]:
                    break
                if stop is not None and stop.is_set():
                    break
                t0 = time.monotonic()
                try:
                    if cli is None:
                        raise RequestFailure("no connection")
                    _, head = cli.predict(x)
                    t1 = time.monotonic()
                    with lock:
                        res.latencies_ms.append((t1 - t0) * 1e3)
                        res.completions_ms.append((t1 - res.t0) * 1e3)
                        res.wall_done.append(t1)
                        res.service_ms.append(float(head.get("service_ms", 0.0)))
                except (OSError, RequestFailure, ValueError):
                    with lock:
                        res.failed += 1
                        if res.failed > budget[0]:
                            abort.set()
                    if cli is not None:
                        cli.close()
                    try:
                        cli = BinaryClient.to(endpoint, timeout_s)
                    except OSError:
                        cli = None
                k += 1
        finally:
            if cli is not None:
                cli.close()

    threads = [threading.Thread(target=run, args=(i,), daemon=True) for i in range(concurrency)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if abort.is_set():
        raise RequestFailure(f"serving load aborted: {res.failed} failed requests")
    return res


def device_loop_load(endpoint: str, batch: int, *, requests_per_call: int = 20,
                     stop: Optional[threading.Event] = None, n_calls: Optional[int] = None,
                     e2e: bool = True, timeout_s: float = 60.0) -> LoadResult:
    """A GPU-bound online-serving load: the worker runs back-to-back requests
    of ``batch`` samples (``bench`` frames; with ``e2e`` every request copies
    its inputs host->device from pinned memory and its outputs back, as a
    serving process would), each request timed on the device with CUDA
    events.  Request latencies therefore include any time the GPU spent on
    another process's kernels in between — what a co-located profiling job
    costs the service.  Completion instants are mapped to the host clock from
    the reply time (the binary-frame clients above measure the whole RPC
    instead, which on a loopback socket is dominated by host copies)."""
    if n_calls is None and stop is None:
        raise ValueError("give n_calls or a stop event")
    from .profiler.clients import make_client
    host, port = split_endpoint(endpoint)
    cli = make_client("grpc-style", host, port, timeout_s)
    res = LoadResult()
    res.t0 = time.monotonic()
    k = 0
    try:
        while (n_calls is None or k < n_calls) and not (stop is not None and stop.is_set()):
            reply = cli.call({"kind": "bench", "batch": batch, "n": requests_per_call,
                              "warmup": 0, "seed": k, "e2e": e2e})
            t_r = time.monotonic()
            if not reply or not reply.get("ok"):
                res.failed += requests_per_call
                raise RequestFailure(f"serving bench failed: {(reply or {}).get('error')}")
            lat, comp = reply["latencies_ms"], reply["completions_ms"]
            end = float(comp[-1])
            for l_ms, c_ms in zip(lat, comp):
                w = t_r - (end - float(c_ms)) / 1e3
                res.latencies_ms.append(float(l_ms))
                res.wall_done.append(w)
                res.completions_ms.append((w - res.t0) * 1e3)
                res.service_ms.append(float(l_ms))
            k += 1
    finally:
        cli.close()
    return res


class DynamicBatcher:
    """Merge concurrent requests into one forward.

    ``submit(x)`` blocks until the merged forward containing ``x`` has run and
    returns (its output rows, service ms of the merged forward, merged batch).
    The first queued request opens a window of ``timeout_ms``; the window
    closes early once ``max_batch`` samples are queued.  Requests are never
    split, so one request larger than ``max_batch`` runs alone."""

    def __init__(self, forward: Callable[[np.ndarray], np.ndarray], max_batch: int,
                 timeout_ms: float = 2.0):
        if max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        self.forward = forward
        self.max_batch = max_batch
        self.timeout_s = timeout_ms / 1e3
        self._cv = threading.Condition()
        self._queue: list = []
        self._halt = False
        self.merged_batches: list[int] = []
        self._thread = threading.Thread(target=self._loop, daemon=True, name="batcher")
        self._thread.start()

    def submit(self, x: np.ndarray):
        slot = {"x": x, "done": threading.Event()}
        with self._cv:
            self._queue.append(slot)
            self._cv.notify_all()
        slot["done"].wait()
        if "error" in slot:
            raise slot["error"]
        return slot["y"], slot["ms"], slot["merged"]

    def close(self) -> None:
        with self._cv:
            self._halt = True
            self._cv.notify_all()
        self._thread.join(timeout=5)

    def _take(self) -> list:
        with self._cv:
            while not self._queue and not self._halt:
                self._cv.wait()
            if self._halt:
                return []
            deadline = time.monotonic() + self.timeout_s
            while True:
                n = sum(s["x"].shape[0] for s in self._queue)
                left = deadline - time.monotonic()
                if n >= self.max_batch or left <= 0:
                    break
                self._cv.wait(left)
            take, total = [], 0
            while self._queue:
                b = self._queue[0]["x"].shape[0]
                if take and total + b > self.max_batch:
                    break
                take.append(self._queue.pop(0))
                total += b
            return take

    def _loop(self) -> None:
        while True:
            take = self._take()
            if not take:
                return
            try:
                x = np.concatenate([s["x"] for s in take]) if len(take) > 1 else take[0]["x"]
                t0 = time.perf_counter()
                y = self.forward(x)
                ms = (time.perf_counter() - t0) * 1e3
                self.merged_batches.append(x.shape[0])
                off = 0
                for s in take:
                    b = s["x"].shape[0]
                    s["y"], s["ms"], s["merged"] = y[off:off + b], ms, x.shape[0]
                    off += b
            except Exception as exc:   # delivered to every waiting request
                for s in take:
                    s["error"] = exc
            for s in take:
                s["done"].set()


def slo_report(res: LoadResult, slo_ms: float, windows: list[tuple[str, float, float]]) -> dict:
    """p50/p99 and SLO verdict per named wall-clock window."""
    out = {}
    for name, a, b in windows:
        n = res.count(a, b)
        p99 = res.p(99, a, b)
        out[name] = {"requests": n, "p50_ms": round(res.p(50, a, b), 4),
                     "p99_ms": round(p99, 4), "slo_ms": slo_ms,
                     "slo_held": bool(n > 0 and p99 <= slo_ms)}
    return out
