"""Multi-GPU profile sweeps: the controller -> profiler glue the reference
lacks (SURVEY.md §3.2 "[absent glue]", §8f rank 4) and the sharding plan for
process-per-GPU runs (§8e).

Two ways to spread a sweep (config C4: 5 models x 9 batch sizes) over GPUs,
both without any data-path collective (cells are independent):

* ``ControllerSweep`` — one host process, one long-lived b200 worker per
  (variant, GPU) (model affinity), the idle-aware ``Controller`` granting
  cells to idle GPUs from telemetry snapshots (per-device concurrency, LPT by
  FLOP cost).  Results land in the jobs exactly as ``Profiler.run_cell`` would
  record them.
* ``lpt_partition`` / ``shard_for_rank`` — a deterministic static partition
  for torchrun-style process-per-GPU runs: rank r executes its shard locally,
  and only the small ``ProfilingResult`` documents are gathered to rank 0
  (``gather_results``, host-side, via torch.distributed object gather).
"""

from __future__ import annotations

import heapq
import threading
import time
from typing import Callable, Optional

from .controller import Controller, ControllerConfig
from .profiler.types import Cell, ProfilingJob, ProfilingResult, is_pool
from .telemetry import DeviceSnapshot, DeviceStats

DEFAULT_SETUP_S = 0.05


def cell_cost(flops_per_sample: float, cell: Cell, requests: int, warmup: int,
              tflops: float = 800.0, setup_s: float = DEFAULT_SETUP_S) -> float:
    """Seconds a cell should take: FLOPs x batch x (n + warmup) at a sustained
    rate, plus a fixed per-cell setup (graph capture, RPC)."""
    return flops_per_sample * cell.batch_size * (requests + warmup) / (tflops * 1e12) + setup_s


def lpt_partition(items: list, cost: Callable[[object], float], k: int) -> list[list]:
    """Longest-processing-time-first greedy partition into k bins (stable)."""
    bins: list[list] = [[] for _ in range(k)]
    heap = [(0.0, i) for i in range(k)]
    heapq.heapify(heap)
    for it in sorted(items, key=lambda x: -cost(x)):
        load, i = heapq.heappop(heap)
        bins[i].append(it)
        heapq.heappush(heap, (load + cost(it), i))
    return bins


def shard_for_rank(units: list, cost: Callable[[object], float], rank: int, world: int) -> list:
    return lpt_partition(units, cost, world)[rank]


def gather_results(results: list[ProfilingResult], rank: int, world: int) -> list:
    """All ranks' result documents on rank 0 (others get [])."""
    if world == 1:
        return list(results)
    import torch.distributed as dist
    docs = [r.to_doc() for r in results]
    bucket = [None] * world if rank == 0 else None
    dist.gather_object(docs, bucket, dst=0)
    if rank != 0:
        return []
    return [ProfilingResult.from_doc(d) for part in bucket for d in part]


class ControllerSweep:
    """Drive jobs to completion on a set of devices with the Controller.

    ``run_cell(job, cell, device) -> ProfilingResult`` executes one concrete
    cell (the caller wires it to Profiler/worker instances); ``sample()``
    returns device utilisations (NVML in production, synthetic in tests).
    """

    def __init__(self, devices: list[str], run_cell, sample: Optional[Callable[[], dict]] = None,
                 cost_fn=None, config: Optional[ControllerConfig] = None,
                 poll_s: float = 0.002):
        self.devices = list(devices)
        self.run_cell = run_cell
        self.sample = sample or (lambda: {d: 0.0 for d in self.devices})
        self.ctrl = Controller(config or ControllerConfig(max_cells_per_job=None, order="lpt",
                                                          consecutive_samples=1),
                               cost_fn=cost_fn)
        self.poll_s = poll_s
        self.errors: list[str] = []
        self.placements: list[tuple[str, str]] = []

    def _snapshot(self) -> DeviceSnapshot:
        util = self.sample()
        busy = self.ctrl.running_cells()
        # a device running our own cell is reported busy-by-us; the controller
        # subtracts it through note_instance_stats
        return DeviceSnapshot(time.time(), {d: DeviceStats(util.get(d, 0.0) if d not in busy
                                                           else 0.0, 0, 1)
                                            for d in self.devices})

    def run(self, jobs: list[ProfilingJob], timeout_s: float = 3600.0) -> float:
        for j in jobs:
            self.ctrl.submit(j)
        lock = threading.Lock()
        done_q: list[str] = []
        threads: dict[str, threading.Thread] = {}
        t0 = time.perf_counter()

        def worker(dev: str, job: ProfilingJob, cell: Cell):
            concrete = cell.on(dev) if is_pool(cell.device) else cell
            try:
                res = self.run_cell(job, concrete, dev)
                with lock:
                    job.results.append(res)
                    job.completed_cells.add(cell.key())
            except Exception as exc:   # a failed cell is recorded, never retried
                with lock:
                    job.completed_cells.add(cell.key())
                    job.failed_cells[cell.key()] = str(exc)
                    self.errors.append(f"{cell.key()}@{dev}: {exc}")
            finally:
                with lock:
                    done_q.append(dev)

        while True:
            with lock:
                finished = list(done_q)
                done_q.clear()
            for dev in finished:
                self.ctrl.note_cell_done(dev)
                threads.pop(dev, None)
            if all(j.is_done() for j in jobs) and not threads:
                break
            if time.perf_counter() - t0 > timeout_s:
                raise TimeoutError("sweep did not finish")
            self.ctrl.on_snapshot(self._snapshot())
            for act in self.ctrl.tick():
                if act.kind == "start_cell":
                    job = self.ctrl.job(act.job_id)
                    self.placements.append((act.cell.key(), act.device))
                    th = threading.Thread(target=worker, args=(act.device, job, act.cell),
                                          daemon=True)
                    threads[act.device] = th
                    th.start()
            for j in jobs:
                if j.is_done() and j.state != "completed":
                    j.state = "completed" if j.results else "failed"
            time.sleep(self.poll_s)
        return time.perf_counter() - t0
