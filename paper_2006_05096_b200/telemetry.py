"""Device telemetry for the controller and the profiler's resource trace.

Restates the reference's provider interface (pkg/src/modelci/telemetry/
providers.py:25-173, sampler.py:23-183): ``DeviceProvider.sample() ->
{device: DeviceStats}`` raising ProviderFailure, snapshots flagged stale on
provider failure, bounded drop-oldest subscriptions, per-instance stats.

New: ``NvmlProvider`` reports ``gpu:0`` .. ``gpu:N-1`` (utilisation =
``nvmlDeviceGetUtilizationRates().gpu / 100``, memory used/total), and GPU
instances are sampled through NVML per-process memory and SM utilisation, so
the reference's "GPU memory usage" and "GPU computation utilization"
indicators (SPEC open question) are finally measured on a GPU.
"""

from __future__ import annotations

import logging
import queue
import threading
import time
from abc import ABC, abstractmethod
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Iterator, Optional

from .errors import NotFound, ProviderFailure

log = logging.getLogger(__name__)


@dataclass
class DeviceStats:
    utilization: float
    memory_used: int
    memory_total: int

    def to_doc(self) -> dict:
        return {"utilization": self.utilization, "memory_used": self.memory_used,
                "memory_total": self.memory_total}


@dataclass
class DeviceSnapshot:
    timestamp: float
    devices: dict = field(default_factory=dict)
    stale: bool = False

    def to_doc(self) -> dict:
        return {"timestamp": self.timestamp,
                "devices": {d: s.to_doc() for d, s in self.devices.items()},
                "stale": self.stale}


@dataclass
class InstanceStats:
    instance_id: str
    timestamp: float
    cpu_fraction: float      # share of the instance's device (CPU or GPU) in [0, 1]
    memory_bytes: int
    net_rx_bytes: int = 0
    net_tx_bytes: int = 0

    def to_doc(self) -> dict:
        return {"instance_id": self.instance_id, "timestamp": self.timestamp,
                "cpu_fraction": self.cpu_fraction, "memory_bytes": self.memory_bytes,
                "net_rx_bytes": self.net_rx_bytes, "net_tx_bytes": self.net_tx_bytes}


class DeviceProvider(ABC):
    @abstractmethod
    def sample(self) -> dict:
        """Current stats of every device this provider knows."""


class HostProvider(DeviceProvider):
    """Host CPU as ``cpu:0`` (providers.py:79-97)."""

    def __init__(self):
        import psutil
        self._ps = psutil
        psutil.cpu_percent(interval=None)

    def sample(self) -> dict:
        try:
            util = self._ps.cpu_percent(interval=None) / 100.0
            mem = self._ps.virtual_memory()
        except OSError as exc:
            raise ProviderFailure(f"host sampling failed: {exc}") from exc
        return {"cpu:0": DeviceStats(min(max(util, 0.0), 1.0), int(mem.used), int(mem.total))}


class SyntheticProvider(DeviceProvider):
    """Scripted ``(t_ms, device, util, used, total)`` events against an
    injectable clock (providers.py:100-131) — the controller's test fake."""

    def __init__(self, events, clock=time.monotonic):
        self.events = sorted(events, key=lambda e: e[0])
        self._clock = clock
        self._t0 = clock()

    @classmethod
    def from_file(cls, path, clock=time.monotonic) -> "SyntheticProvider":
        evs = []
        for line in Path(path).read_text().splitlines():
            line = line.strip()
            if line and not line.startswith("#"):
                t, dev, u, used, total = line.split()
                evs.append((float(t), dev, float(u), int(used), int(total)))
        return cls(evs, clock=clock)

    def elapsed_ms(self) -> float:
        return (self._clock() - self._t0) * 1000.0

    def sample(self) -> dict:
        now = self.elapsed_ms()
        state = {}
        for t, dev, u, used, total in self.events:
            if t <= now:
                state[dev] = DeviceStats(u, used, total)
        return state


class NvmlProvider(DeviceProvider):
    """Every visible GPU as ``gpu:<index>`` through NVML."""

    def __init__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
        except Exception as exc:   # no driver / no library
            raise ProviderFailure(f"NVML unavailable: {exc}") from exc
        self._nv = pynvml
        self._handles = [pynvml.nvmlDeviceGetHandleByIndex(i)
                         for i in range(pynvml.nvmlDeviceGetCount())]
        self._last_ts: dict[int, int] = {}

    def device_count(self) -> int:
        return len(self._handles)

    def sample(self) -> dict:
        out = {}
        try:
            for i, h in enumerate(self._handles):
                u = self._nv.nvmlDeviceGetUtilizationRates(h)
                m = self._nv.nvmlDeviceGetMemoryInfo(h)
                out[f"gpu:{i}"] = DeviceStats(u.gpu / 100.0, int(m.used), int(m.total))
        except self._nv.NVMLError as exc:
            raise ProviderFailure(f"NVML sampling failed: {exc}") from exc
        return out

    def compute_pids(self, index: int) -> set:
        """Pids holding a compute context on GPU `index` (NVML shares the
        host PID namespace here: tools/nvml_probe.py saw the load's own pid)."""
        try:
            return {p.pid for p in self._nv.nvmlDeviceGetComputeRunningProcesses(
                self._handles[index])}
        except self._nv.NVMLError as exc:
            raise ProviderFailure(f"NVML process list failed: {exc}") from exc

    def process_stats(self, index: int, pid: int) -> tuple[float, int]:
        """(SM share in [0,1], used GPU memory bytes) of `pid` on GPU `index`."""
        h = self._handles[index]
        mem = 0
        try:
            for p in self._nv.nvmlDeviceGetComputeRunningProcesses(h):
                if p.pid == pid and p.usedGpuMemory:
                    mem = int(p.usedGpuMemory)
        except self._nv.NVMLError:
            pass
        util = None
        try:
            last = self._last_ts.get(index, 0)
            samples = self._nv.nvmlDeviceGetProcessUtilization(h, last)
            for s in samples:
                self._last_ts[index] = max(self._last_ts.get(index, 0), s.timeStamp)
                if s.pid == pid:
                    util = s.smUtil / 100.0
        except self._nv.NVMLError:
            pass
        if util is None:   # per-process accounting unavailable: device-wide figure
            util = self._nv.nvmlDeviceGetUtilizationRates(h).gpu / 100.0
        if mem == 0:       # pid not visible (PID namespace): device-wide memory in use
            mem = int(self._nv.nvmlDeviceGetMemoryInfo(h).used)
        return min(max(util, 0.0), 1.0), mem


class ProcessStatsReader:
    """CPU share and RSS of a host process (providers.py:134-173)."""

    def __init__(self):
        import psutil
        self._ps = psutil
        self._procs: dict = {}
        self._ncpu = psutil.cpu_count() or 1

    def read(self, pid: int) -> tuple[float, int, int, int]:
        ps = self._ps
        try:
            proc = self._procs.get(pid)
            if proc is None or not proc.is_running():
                proc = ps.Process(pid)
                proc.cpu_percent(interval=None)
                self._procs[pid] = proc
            with proc.oneshot():
                cpu = proc.cpu_percent(interval=None) / 100.0 / self._ncpu
                rss = proc.memory_info().rss
                rx = tx = 0
                try:
                    io = proc.io_counters()
                    rx, tx = getattr(io, "read_chars", 0), getattr(io, "write_chars", 0)
                except (ps.AccessDenied, AttributeError, OSError):
                    pass
            return min(cpu, 1.0), rss, rx, tx
        except (ps.NoSuchProcess, ps.ZombieProcess) as exc:
            self._procs.pop(pid, None)
            raise ProviderFailure(f"process {pid} gone: {exc}") from exc
        except ps.Error as exc:
            raise ProviderFailure(f"cannot sample pid {pid}: {exc}") from exc


class Subscription:
    """Bounded snapshot stream; the producer drops the oldest entry rather
    than block (sampler.py:23-57)."""

    def __init__(self, interval_ms: int, maxsize: int = 16):
        self.interval_ms = interval_ms
        self._q: queue.Queue = queue.Queue(maxsize=maxsize)
        self._last_push = 0.0
        self._closed = threading.Event()

    def push(self, snap: DeviceSnapshot) -> None:
        while True:
            try:
                self._q.put_nowait(snap)
                return
            except queue.Full:
                try:
                    self._q.get_nowait()
                except queue.Empty:
                    pass

    def get(self, timeout: Optional[float] = None) -> Optional[DeviceSnapshot]:
        try:
            return self._q.get(timeout=timeout)
        except queue.Empty:
            return None

    def __iter__(self) -> Iterator[DeviceSnapshot]:
        while not self._closed.is_set():
            s = self.get(timeout=0.25)
            if s is not None:
                yield s

    def close(self) -> None:
        self._closed.set()


class Telemetry:
    """Sampling loop + instance stats (sampler.py:60-183)."""

    def __init__(self, provider: DeviceProvider, interval_ms: int = 1000):
        self.provider = provider
        self.interval_ms = interval_ms
        self._latest: Optional[DeviceSnapshot] = None
        self._lock = threading.Lock()
        self._subs: list[Subscription] = []
        self._halt = threading.Event()
        self._thread: Optional[threading.Thread] = None
        self._procs: Optional[ProcessStatsReader] = None
        self.instance_pid_resolver: Optional[Callable[[str], Optional[int]]] = None
        self.instance_device_resolver: Optional[Callable[[str], Optional[str]]] = None
        self._instance_stats: dict = {}

    def sample_devices(self) -> DeviceSnapshot:
        try:
            snap = DeviceSnapshot(time.time(), self.provider.sample())
        except ProviderFailure as exc:
            log.warning("device provider failed: %s", exc)
            with self._lock:
                prev = self._latest
            snap = DeviceSnapshot(time.time(), dict(prev.devices) if prev else {}, stale=True)
        with self._lock:
            self._latest = snap
        return snap

    def latest(self) -> Optional[DeviceSnapshot]:
        with self._lock:
            return self._latest

    def device_ids(self) -> list[str]:
        s = self.latest()
        return sorted(s.devices) if s else []

    def subscribe(self, interval_ms: Optional[int] = None, maxsize: int = 16) -> Subscription:
        iv = self.interval_ms if interval_ms is None else interval_ms
        if iv < 10:
            raise ValueError("subscription interval must be >= 10 ms")
        sub = Subscription(iv, maxsize)
        with self._lock:
            self._subs.append(sub)
        return sub

    def unsubscribe(self, sub: Subscription) -> None:
        sub.close()
        with self._lock:
            if sub in self._subs:
                self._subs.remove(sub)

    def start(self) -> None:
        if self._thread is None:
            self._halt.clear()
            self._thread = threading.Thread(target=self._run, name="telemetry", daemon=True)
            self._thread.start()

    def stop(self) -> None:
        self._halt.set()
        if self._thread is not None:
            self._thread.join(timeout=5)
            self._thread = None

    def _run(self) -> None:
        while not self._halt.is_set():
            snap = self.sample_devices()
            now = time.monotonic()
            with self._lock:
                subs = list(self._subs)
                cadence = min([self.interval_ms] + [s.interval_ms for s in subs]) / 1000.0
            for s in subs:
                if now - s._last_push >= s.interval_ms / 1000.0 * 0.99:
                    s.push(snap)
                    s._last_push = now
            self._halt.wait(cadence)

    def sample_instance(self, instance_id: str) -> InstanceStats:
        if self.instance_pid_resolver is None:
            raise NotFound("no execution backend wired for instance stats")
        pid = self.instance_pid_resolver(instance_id)
        if pid is None:
            self._instance_stats.pop(instance_id, None)
            raise NotFound(f"no live instance {instance_id}")
        dev = self.instance_device_resolver(instance_id) if self.instance_device_resolver \
            else None
        if dev and dev.startswith("gpu:") and isinstance(self.provider, NvmlProvider):
            frac, mem = self.provider.process_stats(int(dev.split(":")[1]), pid)
            st = InstanceStats(instance_id, time.time(), frac, mem)
        else:
            if self._procs is None:
                self._procs = ProcessStatsReader()
            cpu, rss, rx, tx = self._procs.read(pid)
            st = InstanceStats(instance_id, time.time(), cpu, rss, rx, tx)
        self._instance_stats[instance_id] = st
        return st

    def latest_instance_stats(self, instance_id: str) -> Optional[InstanceStats]:
        return self._instance_stats.get(instance_id)
