#!/usr/bin/env python
"""Benchmark of the B200 profiling hot path (the driver's contract).

One step = one pass of the hot path over one batch: a ResNet-50 bf16 forward
at batch 256 (BASELINE.json configs[1], the largest single-GPU profile cell),
replayed from a CUDA graph inside libb2 with inputs resident in HBM, timed
with CUDA events (``b2_bench``).  ``e2e`` is the same metric through the
C-ABI call with HOST buffers (``b2_bench_e2e``: pinned H2D of the fp32 input
batch, forward, D2H of the logits, every step; the copies of neighbouring steps
overlap the forward on separate streams, as a serving pipeline would).

Multi-GPU (torchrun): one process per GPU, each runs its own replica of the
step (the sweep shards by cell with no data-path collective: "scaling": weak);
a barrier + max-over-ranks brackets the timed region.  ``sweep_c4`` is the
north star's multi-GPU quantity: the C4 profile sweep (5 models x 9 batch
sizes) partitioned over the ranks (request-sharded heavy cells, setup-aware
LPT, no collective but the final gather of sample documents), wall time max
over ranks.

``--impl reference`` times the CPU implementation of the path (the numpy
oracle port of the forward, oracle/plan_ref.py, on all host cores) on a
bounded sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "samples/s & p50/p99 latency per batch size; profile-sweep wall time 1-8 GPU"
UNIT = "samples/s"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["_source"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "_source": "fallback"}


class ClockSampler:
    """SM clock / clock-event (throttle) reasons sampled DURING a timed region:
    NVML polled every 2 ms in a thread (a 20-step ResNet-50 region lasts
    ~60 ms, one nvidia-smi call ~50-100 ms), nvidia-smi as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows: list[tuple] = []     # (sm_mhz, max_mhz, [4 reason flags], util %)
        self.source = "nvml"
        self._halt = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run_nvml(self) -> bool:
        try:
            import pynvml as N
            N.nvmlInit()
            h = None
            try:   # the CUDA device this process runs on (NVML ignores CUDA_VISIBLE_DEVICES)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                h = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = None
            if h is None:
                h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
        except Exception:
            return False
        try:
            while not self._halt.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                u = N.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append((float(sm), float(mx), [bool(r & b) for b in bits], int(u)))
                self._halt.wait(0.002)
        finally:
            try:
                N.nvmlShutdown()
            except Exception:
                pass
        return True

    def _run(self):
        if self._run_nvml():
            return
        self.source = "nvidia-smi"
        while not self._halt.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout
                for line in out.strip().splitlines():
                    c = [x.strip() for x in line.split(",")]
                    self.rows.append((float(c[0]) if c[0].replace(".", "").isdigit() else None,
                                      float(c[1]) if c[1].replace(".", "").isdigit() else None,
                                      [c[2 + i] == "Active" for i in range(4)],
                                      int(c[6]) if c[6].isdigit() else 0))
            except Exception:
                return
            self._halt.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._halt.set()
        self._t.join(timeout=6)

    @staticmethod
    def summary_of(samplers) -> dict:
        rows = [r for s in samplers for r in s.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [r for r in rows if r[3] > 0] or rows
        sm = [r[0] for r in busy if r[0] is not None]
        reasons = sorted({ClockSampler.NAMES[i] for r in busy for i in range(4) if r[2][i]})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": rows[0][1], "reasons": reasons, "samples": len(busy),
                "source": samplers[0].source,
                "regions": "device-timed and e2e-timed regions"}

    def summary(self) -> dict:
        return self.summary_of([self])


def build_plan(model: str, dtype: int) -> bytes:
    from paper_2006_05096_b200 import zoo
    return zoo.build_plan(model, dtype, seed=0)


def cpu_baseline(model: str, plan_bytes: bytes, seconds: float = 12.0, batch: int = 4) -> dict:
    """The oracle port (numpy fp32 forward, all host threads) on a bounded
    sample: `batch`-sample forwards repeated for ~`seconds`."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np
    import plan_ref
    from paper_2006_05096_b200 import plan as P
    pl = P.decode(plan_bytes)
    x = plan_ref.make_inputs(pl, batch, 0)
    plan_ref.forward(pl, x, np.float32)   # warm-up (BLAS threads, page-in)
    n = 0
    t0 = time.perf_counter()
    while True:
        plan_ref.forward(pl, x, np.float32)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 50:
            break
    out = {"value": n * batch / el, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
           "sample": f"{n} x {model} fp32 forwards of batch {batch} (numpy oracle, "
                     f"{el:.1f} s)"}
    tc = torch_cpu_forward(model, batch, seconds / 2)
    if tc:
        out["torch_cpu_fp32"] = tc
    return out


def torch_cpu_forward(model: str, batch: int, seconds: float) -> dict | None:
    """BASELINE.md §2(ii)'s compute baseline beside the port: the torchvision /
    transformers fp32 forward on all host threads (random init, same shapes),
    bounded to ~`seconds`.  Supplementary: the reference itself computes
    nothing, the oracle port above is the contract's cpu_baseline."""
    try:
        import torch
        torch.set_num_threads(os.cpu_count())
        if model == "bert":
            from transformers import BertConfig, BertModel
            net = BertModel(BertConfig()).eval()
            x = torch.randint(0, 30522, (batch, 128))
        else:
            import torchvision
            net = getattr(torchvision.models, model)(weights=None).eval()
            x = torch.randn(batch, 3, 224, 224)
        with torch.inference_mode():
            net(x)
            n, t0 = 0, time.perf_counter()
            while True:
                net(x)
                n += 1
                el = time.perf_counter() - t0
                if el >= seconds or n >= 50:
                    break
        return {"value": round(n * batch / el, 2), "unit": UNIT, "threads": os.cpu_count(),
                "sample": f"{n} x torch CPU fp32 {model} forwards of batch {batch} ({el:.1f} s)"}
    except Exception as e:  # torchvision / transformers missing on the box: say so
        return {"unavailable": f"{type(e).__name__}: {e}"[:160]}


def roofline(plan, model: str, batch: int, ms_per_step: float, pk: dict) -> dict:
    """Tensor roofline of the dominant kernel family — the tcgen05 conv/GEMM
    kernels (tc_gemm, tc_gemm2 CTA pair, conv_band(_pair), stem_pool,
    chain_gemm), which run every conv/linear op of the forward.

    achieved = algorithmic FLOPs of one forward (the plan's flops_per_sample,
    true channel counts: 8.178 GFLOP/sample for ResNet-50) x
    batch, divided by the time those kernels take per step = the CUDA-graph
    step time measured in this run x their share of the forward in the
    committed ncu launch list (profiles/ncu_traffic.json from
    tools/ncu_traffic_json.py, same model/batch).
    ``frac_whole_step`` charges the whole step (every kernel) instead.  Peak =
    the measured BURST bf16 figure (a ~3 ms forward replayed for < 1 s runs
    at boost clocks, not under the sustained power cap)."""
    flops = plan.flops_per_sample * batch
    peak = pk.get("bf16_tflops", 1590.0)
    share, traffic, launches, src = None, None, None, None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        tj = json.loads(tp.read_text())
        if tj.get("model", "resnet50") == model and int(tj.get("batch", 256)) == batch:
            share = tj.get("tcgen05_time_share_ncu")
            traffic = tj.get("tcgen05_bytes_per_launch")
            launches = tj.get("tcgen05_launches_per_forward")
            src = tj.get("source")
    t_ms = ms_per_step * (share if share else 1.0)
    achieved = flops / (t_ms / 1e3) / 1e12
    whole = flops / (ms_per_step / 1e3) / 1e12
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": "tcgen05 conv/GEMM family (tc_gemm, tc_gemm2 CTA pair, conv_band, "
                      "conv_band_pair, stem_pool, chain_gemm): every conv/linear op",
            "flops_per_step": flops, "kernel_ms_per_step": round(t_ms, 4),
            "share_of_step_ncu": share, "launches_per_step": launches,
            "avg_launch_ms": round(t_ms / launches, 5) if launches else None,
            "frac_whole_step": round(whole / peak, 4),
            "frac_of_sustained": round(achieved / pk.get("bf16_tflops_sustained", 1400.0), 4),
            "peak_source": f"MEASURED_PEAKS.json bf16_tflops burst ({pk['_source']})",
            "share_source": src}


def per_op_table(plan, blob: bytes, batch: int, ms_per_step: float, pk: dict,
                 top: int = 12) -> list:
    """Per-op fractions (eager per-op CUDA events, scaled so they sum to the
    graph-replayed step): the costliest ops with their achieved TFLOP/s (or
    GB/s for the memory-bound ones) and fraction of the measured peak."""
    from paper_2006_05096_b200 import plan as P
    pl = P.decode(blob)
    prof = plan.profile_ops(batch, iters=3)
    total = sum(ms for _, ms in prof) or 1.0
    scale = ms_per_step / total
    true_c = {o[P.P_IN_OUT]: o[P.P_IN_C] for o in pl.ops if o.kind == P.OP_INPUT}
    rows = []
    for i, (o, (_, ms)) in enumerate(zip(pl.ops, prof)):
        ms *= scale
        if ms <= 0.0005:
            continue    # fused into a neighbour (its time is the neighbour's)
        fl = 0.0
        if o.kind == P.OP_CONV:
            cin = min(o[P.P_CV_CIN], true_c.get(o[P.P_CV_IN], o[P.P_CV_CIN]))
            fl = 2.0 * o[P.P_CV_OH] * o[P.P_CV_OW] * o[P.P_CV_COUT] * o[P.P_CV_R] * \
                o[P.P_CV_S] * cin * batch
        elif o.kind == P.OP_LINEAR:
            fl = 2.0 * o[P.P_LN_ROWS] * o[P.P_LN_N] * o[P.P_LN_K] * batch
        r = {"op": i, "name": o.name, "ms": round(ms, 4)}
        if fl:
            tf = fl / (ms / 1e3) / 1e12
            r.update(tflops=round(tf, 1), frac=round(tf / pk.get("bf16_tflops", 1590.0), 3))
        rows.append(r)
    rows.sort(key=lambda r: -r["ms"])
    return rows[:top]


C4_MODELS = ("mlp", "mobilenet_v2", "resnet50", "bert", "vgg16")
C4_BATCHES = (1, 2, 4, 8, 16, 32, 64, 128, 256)
# algorithmic FLOPs per sample (the plans' own flops_per_sample)
C4_FLOPS = {"mlp": 406528, "mobilenet_v2": 601548544, "resnet50": 8178368512,
            "bert": 22348431360, "vgg16": 30940528640}


def sweep_leg(rank: int, world: int, barrier, max_over_ranks, requests: int = 100,
              warmup: int = 10) -> dict:
    """The C4 profile sweep (BASELINE configs[3]: 5 models x 9 batch sizes,
    n=100 requests + 10 warm-up per cell, device-timed) over the ranks of
    this job, one process per GPU and no data-path collective: heavy cells
    request-sharded, units partitioned by the setup-aware LPT
    (sweeprun.partitioned_sweep), each rank loading only the models of its
    share and measuring its units with b2_bench; only the samples documents
    are gathered.  Wall time = barrier to barrier, max over ranks, plan
    loading (the per-GPU worker start) included."""
    import numpy as np
    from paper_2006_05096_b200 import plan as P, runtime as R
    from paper_2006_05096_b200.profiler.stats import LatencySamples
    from paper_2006_05096_b200.profiler.types import ProfilingJob, SweepSpec
    from paper_2006_05096_b200.sweeprun import cell_cost, partition_units, run_units
    jobs = [ProfilingJob(f"c4-{m}", m, m, SweepSpec(batch_sizes=list(C4_BATCHES),
                                                    devices=["gpu:*"], backends=["b200"],
                                                    protocols=["grpc-style"],
                                                    requests_per_cell=requests,
                                                    warmup_requests=warmup)) for m in C4_MODELS]
    cost = lambda j, c: cell_cost(C4_FLOPS[j.variant_id], c, c.shard_requests(requests), warmup)
    mine = partition_units(jobs, world, cost, setup_s=lambda j: 1.0)[rank]
    # conversion (register -> convert: model -> plan bytes) happens before a
    # sweep in MLModelCI; only the plan loads (the worker starts) are timed
    blobs = {m: build_plan(m, P.DT_BF16) for m in sorted({j.variant_id for j, _ in mine})}
    plans, busy = {}, [0.0]

    def measure(job, unit):
        m = job.variant_id
        if m not in plans:
            plans[m] = R.Plan(blobs[m], P.DT_BF16)
        lat, comp = plans[m].bench(unit.batch_size, unit.shard_requests(requests), warmup,
                                   seed=unit.shard)
        busy[0] += float(comp[-1]) / 1e3
        return LatencySamples([float(v) for v in lat], [float(v) for v in comp])

    barrier()
    t0 = time.perf_counter()
    results = run_units(jobs, mine, rank, world, measure)
    barrier()
    wall = max_over_ranks(time.perf_counter() - t0)
    dev = max_over_ranks(busy[0])
    for pl in plans.values():
        pl.close()
    out = {"wall_s": round(wall, 3), "gpus": world, "cells": len(results) if rank == 0 else None,
           "busiest_rank_device_s": round(dev, 3),
           "config": "C4: " + ",".join(C4_MODELS) + " x batches 1..256, n=100 + 10 warm-up "
                     "per cell, bf16, request-sharded heavy cells, setup-aware LPT over ranks",
           "timing": "host wall clock, barrier to barrier, max over ranks; plan loads (the "
                     "per-GPU worker starts) inside, model conversion before"}
    if rank == 0:
        out["sharded_cells"] = sorted(f"{r.variant_id}:{r.batch_size}"
                                      for r in results if "," in r.device)
        out["per_cell"] = {f"{r.variant_id}:{r.batch_size}": [round(r.peak_throughput, 1),
                                                              round(r.p50_latency_ms, 4),
                                                              round(r.p99_latency_ms, 4)]
                           for r in results}
    return out


def run_ours(args) -> dict | None:
    rank, local, world = dist_env()
    if world > 1:
        os.environ.setdefault("CUDA_VISIBLE_DEVICES", str(local))
    import numpy as np
    from paper_2006_05096_b200 import plan as P, runtime as R
    dt = P.DT_BF16 if args.dtype == "bf16" else P.DT_FP32
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        pg = dist
    blob = build_plan(args.model, dt)
    plan = R.Plan(blob, dt)
    B, K, W = args.batch, args.steps, args.warmup

    def barrier():
        if pg is not None:
            pg.barrier()

    def max_over_ranks(v: float) -> float:
        if pg is None:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64,
                         device="cuda" if torch.cuda.is_available() else "cpu")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    # device-resident timed region: K graph replays bracketed by CUDA events
    plan.bench(B, 2, 1, seed=1)               # build workspaces + graph outside the region
    barrier()
    with ClockSampler(0 if world > 1 else int(os.environ.get("B2_GPU_INDEX", "0"))) as clk:
        lat, comp = plan.bench(B, K, W, seed=0)
    barrier()
    elapsed_ms = max_over_ranks(float(comp[-1]))
    value = world * K * B / (elapsed_ms / 1e3)
    # end-to-end through the C ABI with host buffers (pinned H2D + D2H per step)
    plan.bench(B, 1, 1, seed=2, e2e=True)
    barrier()
    with ClockSampler(0 if world > 1 else int(os.environ.get("B2_GPU_INDEX", "0"))) as clk_e2e:
        elat, ecomp = plan.bench(B, K, W, seed=0, e2e=True)
    barrier()
    e2e_ms = max_over_ranks(float(ecomp[-1]))
    e2e_value = world * K * B / (e2e_ms / 1e3)
    sweep = None
    if not args.no_c4:
        sweep = sweep_leg(rank, world, barrier, max_over_ranks)
    if rank != 0:
        if pg is not None:
            pg.destroy_process_group()
        return None
    pk = peaks()
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(elapsed_ms / K, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (seeded N(0,1) images; seeded random-init "
                                     "weights, BN calibrated)",
        "config": {"workload": f"{args.model} {args.dtype} profile cell, batch {B} "
                               "(BASELINE configs[1])", "model": args.model,
                   "global_batch": B * world, "seq_len": None,
                   "parallelism": f"replicas x{world} (cells shard, no collective)",
                   "l2": "inputs larger than L2 (fp32 input batch %.0f MB + activations)"
                         % (B * plan.in_elems * 4 / 1e6)},
        "p50_ms": round(float(np.percentile(lat, 50)), 4),
        "p99_ms": round(float(np.percentile(lat, 99)), 4),
        "e2e": {"value": round(e2e_value, 1), "unit": UNIT,
                "h2d_bytes_per_step": int(B * plan.in_elems * 4),
                "d2h_bytes_per_step": int(B * plan.out_elems * 4),
                "ms_per_step": round(e2e_ms / K, 4),
                "p50_ms": round(float(np.percentile(elat, 50)), 4),
                "mode": "b2_bench_e2e: pinned fp32 inputs H2D + forward + logits D2H every step, "
                        "software-pipelined over 3 streams (H2D i+1 and D2H i-1 overlap forward i)"},
        "gpu_launches": int(K * plan.launches_per_forward),
        "clocks": ClockSampler.summary_of([clk, clk_e2e]),
    }
    if sweep is not None:
        line["sweep_c4"] = sweep
    line["roofline"] = roofline(plan, args.model, B, elapsed_ms / K, pk)
    line["roofline"]["per_op"] = per_op_table(plan, blob, B, elapsed_ms / K, pk)
    if not args.no_sweep:
        table = {}
        for b in (1, 2, 4, 8, 16, 32, 64, 128, 256):
            l, c = plan.bench(b, 20, 3, seed=b)
            table[str(b)] = {"samples_s": round(20 * b / (float(c[-1]) / 1e3), 1),
                             "p50_ms": round(float(np.percentile(l, 50)), 4),
                             "p99_ms": round(float(np.percentile(l, 99)), 4)}
        line["per_batch"] = table
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.model, blob)
    if pg is not None:
        pg.destroy_process_group()
    return line


def run_reference(args) -> dict | None:
    rank, _, world = dist_env()
    if rank != 0:
        return None
    from paper_2006_05096_b200 import plan as P
    blob = build_plan(args.model, P.DT_FP32)
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np
    import plan_ref
    pl = P.decode(blob)
    sample = 4   # bounded per-step sample of the batch-256 workload
    x = plan_ref.make_inputs(pl, sample, 0)
    for _ in range(args.warmup):
        plan_ref.forward(pl, x, np.float32)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        plan_ref.forward(pl, x, np.float32)
    el = time.perf_counter() - t0
    value = args.steps * sample / el
    cb = {"value": round(value, 3), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
          "sample": f"{sample} of the {args.batch}-sample batch per step, numpy fp32 oracle "
                    f"forward of {args.model} on all host threads"}
    return {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{args.model} profile cell, batch {args.batch} "
                                   f"(CPU: {sample}-sample bounded step)", "model": args.model,
                       "global_batch": args.batch, "seq_len": None, "parallelism": "cpu"},
            "cpu_baseline": cb,
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--dtype", choices=["bf16", "fp32"], default="bf16")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true",
                    help="skip the C4 profile-sweep wall-time leg (all ranks)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
