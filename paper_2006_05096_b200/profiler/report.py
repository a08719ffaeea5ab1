"""Profile-table export with the reference's fixed CSV schema.

``CSV_COLUMNS`` / ``results_to_csv`` restate pkg/src/modelci/profiler/report.py:16-32
(one row per cell, sorted by (device, backend, protocol, batch), None -> "").
The matplotlib figures of report.py:44-117 are out of scope (matplotlib is
absent from this image); ``results_to_markdown`` gives the same table as text.
Roofline fractions are reported beside the CSV, never inside it.
"""

from __future__ import annotations

import csv
import io

from .types import ProfilingResult

CSV_COLUMNS = [
    "variant_id", "device", "backend", "protocol", "batch_size",
    "peak_throughput", "p50_latency_ms", "p95_latency_ms", "p99_latency_ms",
    "memory_bytes", "utilization", "measured_at", "raw_sample_count",
    "degraded", "resource_scope",
]


def _ordered(results):
    return sorted(results, key=lambda r: (r.device, r.backend, r.protocol, r.batch_size))


def results_to_csv(results: list[ProfilingResult]) -> str:
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=CSV_COLUMNS, lineterminator="\n")
    w.writeheader()
    for r in _ordered(results):
        doc = r.to_doc()
        w.writerow({k: "" if doc[k] is None else doc[k] for k in CSV_COLUMNS})
    return buf.getvalue()


def results_to_markdown(results: list[ProfilingResult]) -> str:
    head = ("| device | backend | batch | samples/s (peak) | p50 ms | p95 ms | p99 ms | "
            "mem MB | util |\n|---|---|---|---|---|---|---|---|---|\n")
    rows = []
    for r in _ordered(results):
        mem = "" if r.memory_bytes is None else f"{r.memory_bytes / 1e6:.0f}"
        util = "" if r.utilization is None else f"{r.utilization:.2f}"
        rows.append(f"| {r.device} | {r.backend} | {r.batch_size} | {r.peak_throughput:,.0f} | "
                    f"{r.p50_latency_ms:.3f} | {r.p95_latency_ms:.3f} | {r.p99_latency_ms:.3f} | "
                    f"{mem} | {util} |")
    return head + "\n".join(rows) + "\n"
