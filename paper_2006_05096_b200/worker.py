"""The B200 executor process: ``python -m paper_2006_05096_b200.worker``.

Drop-in for the reference's serving backend (pkg/src/modelci/mockserve/
__main__.py:18-60, server.py:91-241) behind the same process contract:

* ``--model PATH --protocol rest|grpc-style``; prints ``READY <port>`` once
  listening; exits 2 when the model does not decode (b200-plan, or a toy
  graph which is converted on load); exits 3 when no usable GPU is visible
  (there is no CPU fallback); dies on SIGTERM.
* rest: ``GET /health``; ``POST /predict {"inputs": [[...]]}`` ->
  ``{"outputs", "batch", "service_ms"}`` (400 on an empty batch);
  ``POST /bench`` and ``POST /info`` (new).  TCP_NODELAY is set, removing the
  reference's ~44 ms Nagle floor.
* grpc-style: 4-byte big-endian framed JSON ``{"kind": "health"|"predict"}``
  plus ``predict_bin`` / ``bench`` / ``info`` (wire.py).

``predict`` runs the real forward (libb2 ``b2_forward_host``) instead of
sleeping; ``service_ms`` is the measured device-side request time.  ``bench``
runs a sweep cell's closed loop on the device (libb2 ``b2_bench``) and
returns, with the LatencySamples fields, the cell's own resource trace: per
request the share of device time the forward kept the GPU busy (CUDA-event
latency over the completion interval) and the plan's device memory
(``b2_plan_memory``) — what the reference's ``_ResourceTrace`` samples for a
CPU instance (profiler/sweep.py:51-79), but timed on the device and confined
to the cell.

Reference flags kept: ``--fault-script`` (``<t_ms> health_fail|health_ok``
lines, mockserve/server.py:59-88, __main__.py:26,44) and ``--ready-delay-ms``.
New: ``--max-batch N [--batch-timeout-ms T]`` merges concurrent predict
requests into one forward (online.DynamicBatcher).
"""

from __future__ import annotations

import argparse
import json
import os
import signal
import socketserver
import sys
import threading
import time
from http.server import BaseHTTPRequestHandler, ThreadingHTTPServer
from pathlib import Path

import numpy as np

from . import plan as P
from . import toyformat, wire, zoo
from .errors import LaunchFailure, ModelCIError, PlanFormatError, ToyFormatError

FORMAT_EXIT = 2
NO_DEVICE_EXIT = 3


def load_plan_bytes(data: bytes) -> bytes:
    """b200-plan bytes from a variant file (plans pass through; toy graphs are
    lowered with the toy converter, so a reference toy variant also loads)."""
    return load_plan(data)[0]


def load_plan(data: bytes) -> tuple[bytes, dict]:
    """(plan bytes, plan meta) — decoded once (magic, CRC, tables)."""
    if data[:4] != P.MAGIC:
        graph = toyformat.load_model(data)
        data = zoo.emit_toy(graph, "toy").build(P.DT_FP32)
    # the library's b2_plan_create verifies the CRC; the Python decode only
    # needs the tables (skips a second pass over up to 0.5 GB of weights)
    return data, P.decode(data, verify_crc=False).meta


class FaultScript:
    """Timed health flips: lines of ``<t_ms> health_fail|health_ok``; the state
    at time t is the last action whose timestamp has passed (the reference's
    FaultScript, mockserve/server.py:59-88)."""

    ACTIONS = {"health_fail": False, "health_ok": True}

    def __init__(self, events: list[tuple[float, str]]):
        for _, action in events:
            if action not in self.ACTIONS:
                raise ValueError(f"unknown fault action '{action}'")
        self.events = sorted(events)

    @classmethod
    def from_file(cls, path) -> "FaultScript":
        events = []
        for line in Path(path).read_text().splitlines():
            line = line.strip()
            if line and not line.startswith("#"):
                t_ms, action = line.split()
                events.append((float(t_ms), action))
        return cls(events)

    def healthy_at(self, elapsed_ms: float) -> bool:
        ok = True
        for t_ms, action in self.events:
            if t_ms <= elapsed_ms:
                ok = self.ACTIONS[action]
        return ok


class Executor:
    """Model behaviour shared by both protocols (the MockServer analogue)."""

    def __init__(self, plan_bytes: bytes, dtype: int, meta: dict | None = None,
                 fault_script: FaultScript | None = None, max_batch: int = 0,
                 batch_timeout_ms: float = 2.0):
        from .runtime import Plan
        self.plan = Plan(plan_bytes, dtype)
        self.meta = meta if meta is not None else P.decode(plan_bytes).meta
        self.fault_script = fault_script or FaultScript([])
        self.started = time.monotonic()
        self.batcher = None
        if max_batch > 0:
            from .online import DynamicBatcher
            self.batcher = DynamicBatcher(self.plan.predict, max_batch, batch_timeout_ms)

    def healthy(self) -> bool:
        return self.fault_script.healthy_at((time.monotonic() - self.started) * 1000.0)

    def info(self) -> dict:
        p = self.plan
        return {"ok": True, "in_elems": p.in_elems, "out_elems": p.out_elems,
                "in_kind": p.in_kind, "dtype": p.dtype, "flops_per_sample": p.flops_per_sample,
                "weight_bytes": p.weight_bytes, "launches_per_forward": p.launches_per_forward,
                "model": self.meta.get("model", "")}

    def predict_array(self, x: np.ndarray) -> tuple[np.ndarray, float]:
        if self.batcher is not None:
            out, ms, _ = self.batcher.submit(x)
            return out, ms
        t0 = time.perf_counter()
        out = self.plan.predict(x)
        return out, (time.perf_counter() - t0) * 1000.0

    def predict(self, inputs) -> dict:
        if not isinstance(inputs, list) or not inputs:
            raise ValueError("batch must be a non-empty list of samples")
        x = np.asarray(inputs, dtype=self.plan.in_dtype)
        if x.ndim != 2 or x.shape[1] != self.plan.in_elems:
            raise ValueError(f"samples must have {self.plan.in_elems} elements")
        out, ms = self.predict_array(x)
        return {"outputs": out.tolist(), "batch": int(x.shape[0]), "service_ms": ms}

    def bench(self, req: dict) -> dict:
        batch = int(req.get("batch", 1))
        n = int(req.get("n", 100))
        warm = int(req.get("warmup", 10))
        seed = int(req.get("seed", 0))
        if batch < 1 or n < 1:
            raise ValueError("batch and n must be >= 1")
        lat, comp = self.plan.bench(batch, n, warm, seed, e2e=bool(req.get("e2e", False)))
        mem = self.plan.device_bytes()
        prev = np.concatenate([[0.0], comp[:-1]])
        busy = np.clip(lat / np.maximum(comp - prev, 1e-9), 0.0, 1.0)
        return {"ok": True, "batch": batch, "latencies_ms": lat.tolist(),
                "completions_ms": comp.tolist(),
                "resource_trace": [[float(t), float(b), mem] for t, b in zip(comp, busy)],
                "device_bytes": mem}


class _RestServer(ThreadingHTTPServer):
    daemon_threads = True
    allow_reuse_address = True

    def __init__(self, addr, handler, ex: Executor):
        super().__init__(addr, handler)
        self.ex = ex


class _RestHandler(BaseHTTPRequestHandler):
    protocol_version = "HTTP/1.1"
    disable_nagle_algorithm = True

    def log_message(self, fmt, *args):
        pass

    def _send(self, status: int, payload: dict):
        body = json.dumps(payload).encode()
        self.send_response(status)
        self.send_header("Content-Type", "application/json")
        self.send_header("Content-Length", str(len(body)))
        self.end_headers()
        self.wfile.write(body)

    def do_GET(self):
        if self.path == "/health":
            if self.server.ex.healthy():
                self._send(200, {"status": "ok"})
            else:
                self._send(503, {"status": "unhealthy"})
        else:
            self._send(404, {"error": "not found"})

    def do_POST(self):
        try:
            n = int(self.headers.get("Content-Length", "0"))
            req = json.loads(self.rfile.read(n) or b"{}")
            ex = self.server.ex
            if self.path == "/predict":
                self._send(200, ex.predict(req.get("inputs")))
            elif self.path == "/bench":
                self._send(200, ex.bench(req))
            elif self.path == "/info":
                self._send(200, ex.info())
            else:
                self._send(404, {"error": "not found"})
        except (ValueError, json.JSONDecodeError, ModelCIError) as exc:
            self._send(400, {"ok": False, "error": str(exc)})


class _FrameServer(socketserver.ThreadingTCPServer):
    daemon_threads = True
    allow_reuse_address = True

    def __init__(self, addr, handler, ex: Executor):
        super().__init__(addr, handler)
        self.ex = ex


class _FrameHandler(socketserver.BaseRequestHandler):
    def handle(self):
        ex = self.server.ex
        wire.nodelay(self.request)
        while True:
            try:
                raw = wire.read_frame(self.request)
            except (ConnectionError, ValueError, OSError):
                return
            if raw is None:
                return
            try:
                reply = self._dispatch(ex, raw)
            except (ValueError, json.JSONDecodeError, ModelCIError) as exc:
                reply = json.dumps({"ok": False, "error": str(exc)}).encode()
            try:
                wire.write_frame(self.request, reply)
            except (ConnectionError, OSError):
                return

    @staticmethod
    def _dispatch(ex: Executor, raw: bytes) -> bytes:
        if raw.startswith(wire.BIN_MAGIC):
            head, body = wire.unpack_bin(raw)
            if head.get("kind") != "predict_bin":
                raise ValueError(f"unknown binary kind '{head.get('kind')}'")
            batch = int(head.get("batch", 0))
            x = np.frombuffer(body, dtype=ex.plan.in_dtype)
            if batch < 1 or x.size != batch * ex.plan.in_elems:
                raise ValueError("binary batch does not match the model input size")
            out, ms = ex.predict_array(x.reshape(batch, ex.plan.in_elems))
            return wire.pack_bin({"ok": True, "batch": batch, "out_elems": ex.plan.out_elems,
                                  "service_ms": ms}, out.tobytes())
        msg = json.loads(raw)
        kind = msg.get("kind")
        if kind == "health":
            ok = ex.healthy()
            reply = {"ok": ok, "status": "ok" if ok else "unhealthy"}
        elif kind == "predict":
            reply = dict(ex.predict(msg.get("inputs")), ok=True)
        elif kind == "bench":
            reply = ex.bench(msg)
        elif kind == "info":
            reply = ex.info()
        else:
            reply = {"ok": False, "error": f"unknown kind '{kind}'"}
        return json.dumps(reply).encode()


def serve(ex: Executor, protocol: str, host: str = "127.0.0.1"):
    if protocol == "rest":
        return _RestServer((host, 0), _RestHandler, ex)
    if protocol == "grpc-style":
        return _FrameServer((host, 0), _FrameHandler, ex)
    raise ValueError(f"unknown protocol '{protocol}'")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="b200-worker", description="B200 model executor")
    ap.add_argument("--model", required=True)
    ap.add_argument("--protocol", choices=["rest", "grpc-style"], default="rest")
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--dtype", choices=["auto", "bf16", "fp32"], default="auto",
                    help="execution dtype (auto: the plan header's)")
    ap.add_argument("--fault-script", default=None, help="file of '<t_ms> <action>' lines")
    ap.add_argument("--ready-delay-ms", type=float, default=0.0,
                    help="artificial delay before announcing readiness (for tests)")
    ap.add_argument("--max-batch", type=int, default=0,
                    help="dynamic batching: merge concurrent predicts up to this many samples")
    ap.add_argument("--batch-timeout-ms", type=float, default=2.0,
                    help="dynamic batching: how long the first request waits for company")
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    t_start = time.perf_counter()
    timing = os.environ.get("B2_WORKER_TIMING") == "1"
    try:
        data = Path(args.model).read_bytes()
        t_read = time.perf_counter()
        plan_bytes, meta = load_plan(data)
        t_dec = time.perf_counter()
    except OSError as exc:
        print(f"cannot read model: {exc}", file=sys.stderr)
        return FORMAT_EXIT
    except (PlanFormatError, ToyFormatError) as exc:
        print(f"cannot decode model: {exc}", file=sys.stderr)
        return FORMAT_EXIT
    dtype = {"auto": -1, "bf16": P.DT_BF16, "fp32": P.DT_FP32}[args.dtype]
    try:
        fault = FaultScript.from_file(args.fault_script) if args.fault_script else None
    except (ValueError, OSError) as exc:
        print(f"cannot start: {exc}", file=sys.stderr)
        return FORMAT_EXIT
    try:
        ex = Executor(plan_bytes, dtype, meta, fault_script=fault, max_batch=args.max_batch,
                      batch_timeout_ms=args.batch_timeout_ms)
    except PlanFormatError as exc:
        print(f"cannot load plan: {exc}", file=sys.stderr)
        return FORMAT_EXIT
    except LaunchFailure as exc:
        print(f"no usable device: {exc}", file=sys.stderr)
        return NO_DEVICE_EXIT
    if timing:
        t_ready = time.perf_counter()
        print(f"worker start: read {t_read - t_start:.3f} s, decode {t_dec - t_read:.3f} s, "
              f"plan create {t_ready - t_dec:.3f} s", file=sys.stderr)
    server = serve(ex, args.protocol, args.host)
    if args.ready_delay_ms > 0:
        time.sleep(args.ready_delay_ms / 1000.0)
    # SIGTERM ends the process at once: the driver reclaims the CUDA context
    # and device memory.  A graceful interpreter shutdown (module teardown,
    # context destroy) took 2-3 s per worker, which the profiler's per-job
    # instance teardown (run_sweep) waited for between models.
    signal.signal(signal.SIGTERM, lambda *_: os._exit(0))
    print(f"READY {server.server_address[1]}", flush=True)
    try:
        server.serve_forever(poll_interval=0.05)
    except KeyboardInterrupt:
        pass
    return 0


if __name__ == "__main__":
    sys.exit(main())
