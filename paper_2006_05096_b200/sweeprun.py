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


def plan_shards(jobs: list[ProfilingJob], n_devices: int,
                cost_fn: Callable[[ProfilingJob, Cell], float],
                max_share: float = 0.5, min_requests: int = 10) -> dict:
    """Request-shard the cells that would bound the makespan.

    A pool cell whose cost exceeds ``max_share`` x the ideal per-device load
    (total cost / devices) is split into k shards, k the smallest count that
    brings each shard under that bound, capped by the device count and by
    ``requests_per_cell // min_requests`` (each shard keeps >= 10 timed
    requests, the SweepSpec minimum).  Writes ``job.shard_plan`` and returns
    {(job id, cell key): k} for the cells it split."""
    if n_devices <= 1:
        return {}
    cells = [(j, c) for j in jobs for c in j.remaining_cells() if is_pool(c.device)]
    total = sum(cost_fn(j, c) for j, c in cells)
    bound = max_share * total / n_devices
    out = {}
    for j, c in cells:
        cost = cost_fn(j, c)
        if bound <= 0 or cost <= bound or c.key() in j.shard_plan:
            continue
        k = min(n_devices, max(1, j.sweep.requests_per_cell // min_requests),
                math.ceil(cost / bound))
        if k > 1:
            j.shard_plan[c.key()] = k
            out[(j.id, c.key())] = k
    return out


def fold_units(job: ProfilingJob, measured: list) -> list[ProfilingResult]:
    """Fold measured units of one job into ProfilingResults (rank 0 of a
    partitioned sweep).  ``measured`` = [(unit key, device, LatencySamples)];
    a sharded cell folds once all its shards are present (percentiles over
    the union, peak = max of per-shard peaks), with the devices of its shards
    as the result's device."""
    from .profiler.stats import ShardedSamples, aggregate
    by_base: dict = {}
    for key, dev, samp in measured:
        unit = Cell.from_key(key)
        by_base.setdefault(unit.base().key(), []).append((unit, dev, samp))
    out = []
    for cell in job.sweep.cells():
        parts = by_base.get(cell.key())
        if not parts:
            continue
        k = parts[0][0].shards
        if len(parts) != k:
            continue
        parts.sort(key=lambda p: p[0].shard)
        devs = sorted({d for _, d, _ in parts}, key=lambda d: (len(d), d))
        dev = ",".join(devs)
        samples = parts[0][2] if k == 1 else ShardedSamples([p[2] for p in parts])
        trace = [r for _, _, sm in parts for r in (sm.device_trace or [])]
        res = aggregate(samples, trace, cell.batch_size, variant_id=job.variant_id,
                        device=dev, backend=cell.backend, protocol=cell.protocol,
                        resource_scope=dev)
        job.results.append(res)
        job.completed_cells.add(cell.key())
        out.append(res)
    if job.is_done():
        job.state = "completed" if job.results else "failed"
    return out


def partition_units(jobs: list[ProfilingJob], world: int,
                    cost_fn: Callable[[ProfilingJob, Cell], float],
                    setup_s: Callable[[ProfilingJob], float] | None = None) -> list[list]:
    """The static partition of a torchrun-style sweep: heavy cells
    request-sharded (``plan_shards``), then every remaining work unit
    (job, cell-or-shard) placed by the setup-aware LPT (a rank pays a model's
    load once).  Deterministic, so every rank computes the same one."""
    plan_shards(jobs, world, cost_fn)
    units = [(j, u) for j in jobs for u in j.remaining_units()]
    by_id = {j.id: j for j in jobs}
    return lpt_partition(units, lambda ju: cost_fn(*ju), world,
                         group=(lambda ju: ju[0].id) if setup_s else None,
                         setup=(lambda jid: setup_s(by_id[jid])) if setup_s else None)


def run_units(jobs: list[ProfilingJob], mine: list, rank: int, world: int, measure) -> list:
    """Measure this rank's units (``measure(job, unit) -> LatencySamples``)
    and gather only the samples documents to rank 0, which folds them into
    ProfilingResults (returned on rank 0; [] elsewhere)."""
    docs = []
    for job, unit in mine:
        samp = measure(job, unit)
        docs.append((job.id, unit.key(), f"gpu:{rank}", samp.to_doc()))
    if world > 1:
        import torch.distributed as dist
        bucket = [None] * world if rank == 0 else None
        dist.gather_object(docs, bucket, dst=0)
        if rank != 0:
            return []
        docs = [d for part in bucket for d in part]
    from .profiler.stats import LatencySamples
    out = []
    for job in jobs:
        mine_j = [(k, dev, LatencySamples.from_doc(sd)) for jid, k, dev, sd in docs
                  if jid == job.id]
        out += fold_units(job, mine_j)
    return out


def partitioned_sweep(jobs: list[ProfilingJob], rank: int, world: int, measure,
                      cost_fn: Callable[[ProfilingJob, Cell], float],
                      setup_s: Callable[[ProfilingJob], float] | None = None) -> list:
    """The torchrun-style C4 sweep: one process per GPU, no data-path
    collective — ``partition_units`` then ``run_units`` on this rank's share."""
    mine = partition_units(jobs, world, cost_fn, setup_s)[rank]
    return run_units(jobs, mine, rank, world, measure)


class BusyLedger:
    """Our own device-busy intervals per device (host monotonic clock), for
    self-load exclusion when NVML cannot attribute utilisation per process.

    NVML's device utilisation is the busy share of a trailing window (1/6 s
    to 1 s), so a GPU that just finished one of our cells still reads busy.
    ``share(dev, window)`` is the fraction of the last ``window`` seconds
    covered by our cells on ``dev`` — the part of the NVML figure that is
    ours."""

    def __init__(self, clock=time.monotonic):
        self._clock = clock
        self._iv: dict[str, list] = {}
        self._open: dict[str, float] = {}
        self._lock = threading.Lock()

    def begin(self, dev: str) -> None:
        with self._lock:
            self._open[dev] = self._clock()

    def end(self, dev: str) -> None:
        with self._lock:
            t0 = self._open.pop(dev, None)
            if t0 is not None:
                ivs = self._iv.setdefault(dev, [])
                ivs.append((t0, self._clock()))
                del ivs[:-64]

    def share(self, dev: str, window: float = 1.0) -> float:
        now = self._clock()
        lo = now - window
        with self._lock:
            ivs = list(self._iv.get(dev, []))
            if dev in self._open:
                ivs.append((self._open[dev], now))
        busy = sum(max(0.0, min(b, now) - max(a, lo)) for a, b in ivs)
        return min(1.0, busy / window)


class ControllerSweep:
    """Drive profiling jobs to completion on a set of devices with the
    Controller — the daemon glue the reference specifies but lacks
    (reference controller.py:88-243,
    profiler/sweep.py:193-216).

    Each loop: sample device utilisation (NVML in production, scripted in
    tests) -> ``Controller.on_snapshot`` (with ``note_instance_stats`` = our
    own share of every device running one of our cells) -> ``tick()`` ->
    execute its actions:

    * ``start_cell``: run the unit (cell or request shard) on a thread via
      ``run_cell(job, unit, device)``, which measures and records it (the
      Profiler path persists through the JobStore); a returned result not yet
      recorded (simple runners) is recorded here;
    * ``pause_job``: the device stayed busy with load that is not ours; the
      job stops at the cell boundary (the in-flight cell finishes, no further
      cell goes to that device while it is busy) and is persisted as
      ``paused``;
    * ``resume_job``: a paused job got a cell on an idle device again;
    * ``place_instance``: handed to ``on_place(placement_id, record_id,
      device)`` (a serving deployment on the least-utilised idle GPU).

    Self-load exclusion.  NVML's device utilisation is the busy share of a
    short trailing window and cannot be attributed per process on this
    driver (``nvmlDeviceGetProcessUtilization``: Not Supported, measured by
    tools/nvml_probe.py), but the compute-process list can:

    * a device whose compute processes are all ours (``ours_only(dev)``)
      carries no external load, whatever NVML reads: it is fed 0 and is
      granted its next cell the moment the last one ends;
    * on a device shared with a foreign process, a cell ends with a quiet gap
      (``quiet_s`` > the NVML window, nothing of ours running) followed by a
      clean sample that is entirely external load; it is fed while the cell
      still counts as running with our share 0 (``note_instance_stats``), so
      sustained external load pauses the job at that cell boundary exactly as
      the reference's ``_device_busy_for_pause`` (controller.py:150-156)
      would;
    * otherwise (no process list) our share is the ``BusyLedger`` estimate.

    Devices absent from a sample are absent (never idle)."""

    def __init__(self, devices: list[str], run_cell, sample: Optional[Callable[[], dict]] = None,
                 cost_fn=None, config: Optional[ControllerConfig] = None,
                 poll_s: float = 0.002, sample_interval_s: float = 0.0,
                 ours_only: Optional[Callable[[str], bool]] = None, quiet_s: float = 0.0,
                 jobs_store=None, on_event: Optional[Callable[[str, dict], None]] = None,
                 on_place: Optional[Callable[[str, str, str], None]] = None,
                 util_window_s: float = 0.2, clock=time.monotonic):
        self.devices = list(devices)
        self.run_cell = run_cell
        self.sample = sample or (lambda: {d: 0.0 for d in self.devices})
        self.ctrl = Controller(config or ControllerConfig(max_cells_per_job=None, order="lpt",
                                                          consecutive_samples=1),
                               cost_fn=cost_fn)
        self.poll_s = poll_s
        self.sample_interval_s = sample_interval_s
        self.ours_only = ours_only
        self.quiet_s = quiet_s
        self.jobs_store = jobs_store
        self.on_event = on_event or (lambda kind, payload: None)
        self.on_place = on_place
        self.util_window_s = util_window_s
        self.ledger = BusyLedger(clock)
        self._clock = clock
        self.errors: list[str] = []
        self.placements: list[tuple[str, str]] = []
        self.actions: list[tuple[float, dict]] = []
        self.snapshots: list[tuple[float, dict]] = []
        self.quiet_samples: list[tuple[float, str, float]] = []

    # -- telemetry -------------------------------------------------------------
    @staticmethod
    def _util(v) -> Optional[DeviceStats]:
        if v is None:
            return None
        return v if isinstance(v, DeviceStats) else DeviceStats(float(v), 0, 1)

    def _exclusive(self, dev: str) -> bool:
        try:
            return bool(self.ours_only(dev)) if self.ours_only else False
        except Exception:     # process list unavailable: fall back to the ledger
            return False

    def _snapshot(self, clean: Optional[dict] = None) -> DeviceSnapshot:
        """One snapshot; ``clean`` = {dev: util} measured in a quiet gap
        (entirely external) for devices whose cell is just ending."""
        raw = self.sample()
        running = self.ctrl.running_cells()
        devs = {}
        for d in self.devices:
            if clean and d in clean:
                st = self._util(clean[d])
                self.ctrl.note_instance_stats(d, 0.0)
                devs[d] = st
                continue
            st = self._util(raw.get(d))
            if st is None:
                continue                      # absent, not idle
            if self._exclusive(d):
                if d in running:
                    self.ctrl.note_instance_stats(d, st.utilization)
                    util = st.utilization
                else:
                    util = 0.0
            elif d in running:
                self.ctrl.note_instance_stats(d, self.ledger.share(d, self.util_window_s))
                util = st.utilization
            else:
                util = max(0.0, st.utilization - self.ledger.share(d, self.util_window_s))
            devs[d] = DeviceStats(util, st.memory_used, st.memory_total)
        return DeviceSnapshot(time.time(), devs)

    def _save(self, job: ProfilingJob) -> None:
        if self.jobs_store is not None:
            self.jobs_store.save(job)

    # -- the loop ----------------------------------------------------------------
    def run(self, jobs: list[ProfilingJob], timeout_s: float = 3600.0) -> float:
        for j in jobs:
            self.ctrl.submit(j)
        lock = threading.Lock()
        wake = threading.Event()
        done_q: list[tuple[str, Optional[float]]] = []
        threads: dict[str, threading.Thread] = {}
        t0 = self._clock()

        def worker(dev: str, job: ProfilingJob, unit: Cell):
            self.ledger.begin(dev)
            clean = None
            try:
                res = self.run_cell(job, unit, dev)
                base = unit.base()
                with lock:
                    if res is not None and base.key() not in job.completed_cells:
                        job.results.append(res)
                        job.completed_cells.add(base.key())
                        self._save(job)
            except Exception as exc:   # a failed cell is recorded, never retried
                with lock:
                    base = unit.base()
                    if base.key() not in job.failed_cells:
                        for c in base.split(unit.shards):
                            job.shard_samples.pop(c.key(), None)
                        job.completed_cells.add(base.key())
                        job.failed_cells[base.key()] = str(exc)
                        self._save(job)
                    self.errors.append(f"{unit.key()}@{dev}: {exc}")
            finally:
                self.ledger.end(dev)
                if not self._exclusive(dev):
                    # quiet gap, then a sample that is all external load
                    time.sleep(self.quiet_s)
                    try:
                        st = self._util(self.sample().get(dev))
                        clean = None if st is None else st.utilization
                    except Exception:
                        clean = None
                    if clean is not None:
                        self.quiet_samples.append((self._clock() - t0, dev, clean))
                with lock:
                    done_q.append((dev, clean))
                wake.set()

        last_sample = -1e9
        while True:
            with lock:
                finished = list(done_q)
                done_q.clear()
            cleans = {d: c for d, c in finished if c is not None}
            if cleans:
                # the ending cells still count as running: sustained external
                # load seen in their quiet gap pauses their jobs (tick step 1)
                snap = self._snapshot(clean=cleans)
                self.ctrl.on_snapshot(snap)
                self._execute(self.ctrl.tick(), jobs, threads, worker, t0, lock)
            for dev, _ in finished:
                self.ctrl.note_cell_done(dev)
                threads.pop(dev, None)
            for j in jobs:
                if j.is_done() and j.state not in ("completed", "failed"):
                    j.state = "completed" if j.results else "failed"
                    with lock:
                        self._save(j)
                    self.on_event("job_state", {"job_id": j.id, "state": j.state})
            if all(j.is_done() for j in jobs) and not threads:
                break
            now = self._clock()
            if now - t0 > timeout_s:
                raise TimeoutError("sweep did not finish")
            if finished or now - last_sample >= self.sample_interval_s:
                snap = self._snapshot()
                last_sample = now
                self.snapshots.append((now - t0, {d: s.utilization
                                                  for d, s in snap.devices.items()}))
                del self.snapshots[:-4096]
                self.ctrl.on_snapshot(snap)
            self._execute(self.ctrl.tick(), jobs, threads, worker, t0, lock)
            wake.wait(self.poll_s)
            wake.clear()
        return self._clock() - t0

    def _execute(self, actions, jobs, threads, worker, t0, lock) -> None:
        for act in actions:
            self.actions.append((self._clock() - t0, act.to_doc()))
            if act.kind == "start_cell":
                job = self.ctrl.job(act.job_id)
                self.placements.append((act.cell.key(), act.device))
                th = threading.Thread(target=worker, args=(act.device, job, act.cell),
                                      daemon=True)
                threads[act.device] = th
                th.start()
            elif act.kind in ("pause_job", "resume_job"):
                job = self.ctrl.job(act.job_id)
                with lock:
                    self._save(job)
                self.on_event("job_state", {"job_id": act.job_id, "state": job.state,
                                            "device": act.device, "action": act.kind})
            elif act.kind == "place_instance" and self.on_place is not None:
                self.on_place(act.placement_id, act.job_id, act.device)


class CellRunner:
    """``run_cell`` for ControllerSweep over the real profiler: long-lived
    instances per (variant, device, backend, protocol) — model affinity, a
    GPU loads a model once — and ``Profiler.run_unit`` to measure, aggregate
    and persist (JobStore after every cell / shard, like sweep.py:171-178).
    A failing unit is recorded through ``Profiler.record_cell_failure`` and
    its instance torn down."""

    def __init__(self, profiler):
        self.profiler = profiler
        self._inst: dict = {}
        self._lock = threading.Lock()

    def instance(self, job: ProfilingJob, cell: Cell):
        key = (job.variant_id, cell.device, cell.backend, cell.protocol)
        with self._lock:
            inst = self._inst.get(key)
        inst = self.profiler.ensure_instance(job, cell, inst)
        with self._lock:
            self._inst[key] = inst
        return inst

    def prewarm(self, pairs: list) -> None:
        """Dispatch instances for (job, concrete cell) pairs concurrently."""
        import concurrent.futures as cf
        if not pairs:
            return
        with cf.ThreadPoolExecutor(min(16, len(pairs))) as ex:
            list(ex.map(lambda p: self.instance(*p), pairs))

    def instances_on(self, device: str) -> list:
        with self._lock:
            return [i for (_, d, _, _), i in self._inst.items() if d == device]

    def __call__(self, job: ProfilingJob, unit: Cell, device: str):
        concrete = unit.on(device) if is_pool(unit.device) else unit
        try:
            inst = self.instance(job, concrete)
            return self.profiler.run_unit(job, concrete, inst, key_cell=unit)
        except Exception as exc:
            self.profiler.record_cell_failure(job, unit, str(exc))
            key = (job.variant_id, concrete.device, concrete.backend, concrete.protocol)
            with self._lock:
                inst = self._inst.pop(key, None)
            self.profiler.teardown(inst)
            raise

    def shutdown(self) -> None:
        with self._lock:
            insts = list(self._inst.values())
            self._inst.clear()
        for i in insts:
            self.profiler.teardown(i)


def nvml_hooks(provider, runner: CellRunner, pid_of: Callable[[str], Optional[int]]):
    """``sample`` and ``ours_only`` for ControllerSweep on real GPUs: device
    utilisation from NVML, and "every compute process on this GPU is one of
    our workers (or this process)" from NVML's process list."""
    import os

    def sample() -> dict:
        return provider.sample()

    def ours_only(dev: str) -> bool:
        idx = int(dev.split(":")[1])
        mine = {os.getpid()}
        for inst in runner.instances_on(dev):
            pid = pid_of(inst.id)
            if pid is not None:
                mine.add(pid)
        return provider.compute_pids(idx) <= mine

    return sample, ours_only
