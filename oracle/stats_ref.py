"""Brute-force restatement of the profiler's indicator math (TEST
INFRASTRUCTURE ONLY), following pkg/tests/oracles.py:12-36 and the
definitions in pkg/src/modelci/profiler/stats.py:50-104:

* nearest-rank percentile: sorted sample at 1-based ceil(p * n / 100), with a
  decimal p taken at its decimal value (stats.py:50-69);
* peak throughput: max count of completions in half-open windows
  [t, t + window) anchored at completions, x batch x 1000 / window; the
  whole-run rate when the run is shorter than one window (stats.py:72-104).
"""
from fractions import Fraction
import math


def percentile(samples, p):
    ordered = sorted(samples)
    frac = Fraction(str(p)) if isinstance(p, float) else Fraction(p)
    k = math.ceil(frac * len(ordered) / 100)
    return ordered[k - 1]


def peak_throughput(ts, batch, window_ms=1000):
    ts = sorted(ts)
    dur = ts[-1]
    if dur < window_ms:
        return len(ts) * batch * 1000 / dur
    best = 0
    for start in ts:
        best = max(best, sum(1 for t in ts if start <= t < start + window_ms))
    return best * batch * 1000 / window_ms
