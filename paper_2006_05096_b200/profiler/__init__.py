"""Profiler: sweep types, indicator math, timing loops, sweep execution."""

from .report import CSV_COLUMNS, results_to_csv, results_to_markdown
from .stats import LatencySamples, ResourceSample, aggregate, peak_throughput, percentile
from .types import Cell, ProfilingJob, ProfilingResult, SweepSpec

__all__ = ["CSV_COLUMNS", "Cell", "LatencySamples", "ProfilingJob", "ProfilingResult",
           "ResourceSample", "SweepSpec", "aggregate", "peak_throughput", "percentile",
           "results_to_csv", "results_to_markdown"]
