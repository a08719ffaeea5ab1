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
import math
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


def lpt_partition(items: list, cost: Callable[[object], float], k: int,
                  group: Callable[[object], object] | None = None,
                  setup: Callable[[object], float] | None = None) -> list[list]:
    """Longest-processing-time-first greedy partition into k bins (stable).

    With ``group``/``setup``: a bin pays ``setup(g)`` once for every distinct
    group g it hosts (a model's worker start on a GPU), and each item goes to
    the bin where its completion time -- load + cost + any new setup -- is
    smallest, so cells of one model stay together unless splitting pays."""
    bins: list[list] = [[] for _ in range(k)]
    if group is None or setup is None:
        heap = [(0.0, i) for i in range(k)]
        heapq.heapify(heap)
        for it in sorted(items, key=lambda x: -cost(x)):
            load, i = heapq.heappop(heap)
            bins[i].append(it)
            heapq.heappush(heap, (load + cost(it), i))
        return bins
    # two-level LPT: split each group into as many chunks as its work fills
    # bins of the ideal makespan (total work + one setup per group) / k, then
    # place the chunks (work + setup) longest first on the least-loaded bin
    groups: dict = {}
    for it in items:
        groups.setdefault(group(it), []).append(it)
    work = {g: sum(cost(x) for x in xs) for g, xs in groups.items()}
    target = (sum(work.values()) + sum(setup(g) for g in groups)) / k
    chunks = []
    for g, xs in groups.items():
        n = max(1, min(k, len(xs), math.ceil(work[g] / max(target, 1e-12) - 1e-9)))
        for part in lpt_partition(xs, cost, n):
            if part:
                chunks.append((g, part))
    loads = [0.0] * k
    hosted: list[set] = [set() for _ in range(k)]
    for g, part in sorted(chunks, key=lambda c: -(sum(cost(x) for x in c[1]) + setup(c[0]))):
        i = min(range(k), key=lambda j: loads[j])
        bins[i].extend(part)
        loads[i] += sum(cost(x) for x in part) + (0.0 if g in hosted[i] else setup(g))
        hosted[i].add(g)

    def load(b):
        return sum(cost(x) for x in b) + sum(setup(h) for h in {group(x) for x in b})

    # local search: move single items off the busiest bin while that lowers it
    for _ in range(4 * len(items)):
        lds = [load(b) for b in bins]
        hi = max(range(k), key=lambda j: lds[j])
        best = None
        for x in bins[hi]:
            rest = [y for y in bins[hi] if y is not x]
            for j in range(k):
                if j == hi:
                    continue
                new_max = max(load(rest), load(bins[j] + [x]))
                if new_max < lds[hi] - 1e-9 and (best is None or new_max < best[0]):
                    best = (new_max, x, j)
        if best is None:
            break
        _, x, j = best
        bins[hi] = [y for y in bins[hi] if y is not x]
        bins[j].append(x)
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
