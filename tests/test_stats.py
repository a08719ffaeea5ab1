"""Indicator math parity with the reference (golden vectors generated from
pkg/src/modelci/profiler/stats.py by tests/golden/make_golden.py), plus the
reference tests' known answers and properties (pkg/tests/test_stats.py)."""
import json
import random
from pathlib import Path

import pytest
from hypothesis import given, strategies as st

from paper_2006_05096_b200.errors import EmptySamples
from paper_2006_05096_b200.profiler.stats import (LatencySamples, ResourceSample, aggregate,
                                                  peak_throughput, percentile)
import stats_ref

GOLD = json.loads((Path(__file__).parent / "golden" / "stats_golden.json").read_text())


def test_percentile_matches_reference_golden():
    for case in GOLD["percentile"]:
        assert percentile(case["samples"], case["p"]) == case["out"]


def test_peak_throughput_matches_reference_golden():
    for case in GOLD["peak_throughput"]:
        assert peak_throughput(case["ts"], case["batch"], case["window"]) == case["out"]


def test_aggregate_matches_reference_golden():
    for case in GOLD["aggregate"]:
        r = aggregate(LatencySamples(case["lat"], case["comp"]),
                      [ResourceSample(*t) for t in case["trace"]], case["batch"],
                      variant_id="v", device="gpu:0", backend="b200", protocol="grpc-style",
                      resource_scope="gpu:0")
        d = r.to_doc()
        d.pop("measured_at")
        assert d == case["out"]


def test_known_answers():
    k = GOLD["known"]
    assert peak_throughput([10 * i for i in range(1, 201)], 4) == k["steady"] == 400.0
    assert peak_throughput([500], 1) == k["short"] == 2.0
    assert percentile(list(range(1, 101)), 95) == k["p95_1_100"] == 95
    assert percentile([10, 20, 30], 50) == k["p50_three"] == 20
    assert percentile([5, 5, 5, 5], 50) == 5
    assert percentile([3, 1, 2], 100) == 3


def test_matches_bruteforce_oracle_randomized():
    rng = random.Random(0xC0FFEE)
    for _ in range(1000):
        s = [rng.randint(-1000, 1000) for _ in range(rng.randint(1, 60))]
        p = rng.randint(1, 100)
        assert percentile(s, p) == stats_ref.percentile(s, p)
    rng = random.Random(0xBEEF)
    for _ in range(500):
        ts = [rng.randint(1, 4000) for _ in range(rng.randint(1, 80))]
        b, w = rng.randint(1, 16), rng.choice([250, 500, 1000, 2000])
        assert peak_throughput(ts, b, w) == stats_ref.peak_throughput(ts, b, w)


def test_errors():
    with pytest.raises(EmptySamples):
        percentile([], 50)
    with pytest.raises(ValueError):
        percentile([1], 0)
    with pytest.raises(EmptySamples):
        peak_throughput([], 1)
    with pytest.raises(EmptySamples):
        aggregate(LatencySamples([], [], failed=3), [], 1, variant_id="v", device="gpu:0",
                  backend="b", protocol="rest")


def test_empty_trace_degrades():
    r = aggregate(LatencySamples([1.0] * 10, [float(i + 1) for i in range(10)]), [], 1,
                  variant_id="v", device="gpu:0", backend="b200", protocol="rest")
    assert r.degraded and r.memory_bytes is None and r.utilization is None


@given(st.lists(st.integers(-10**6, 10**6), min_size=1, max_size=50), st.integers(1, 99),
       st.integers(2, 100))
def test_monotone_in_p(samples, a, b):
    lo, hi = min(a, b), max(a, b)
    assert percentile(samples, lo) <= percentile(samples, hi)


def test_sharded_cell_union_latency_and_max_peak():
    """A request-sharded cell: latencies are the union of the shards', peak
    throughput the max of the per-shard peaks (never the pooled completions,
    which would report k GPUs' combined rate)."""
    from paper_2006_05096_b200.profiler.stats import ShardedSamples, peak_throughput
    a = LatencySamples([10.0] * 50, [10.0 * (i + 1) for i in range(50)])          # 100 req/s
    b = LatencySamples([12.0] * 50, [12.0 * (i + 1) for i in range(50)], failed=1)
    sh = ShardedSamples([a, b])
    u = sh.union()
    assert sorted(u.latencies_ms) == sorted(a.latencies_ms + b.latencies_ms) and u.failed == 1
    assert sh.peak_throughput(4) == max(peak_throughput(a.completions_ms, 4),
                                        peak_throughput(b.completions_ms, 4)) == 400.0
    pooled = peak_throughput(sorted(a.completions_ms + b.completions_ms), 4)
    assert pooled > 600.0                       # what naive pooling would claim
    r = aggregate(sh, [], 4, variant_id="v", device="gpu:0", backend="b200", protocol="rest")
    assert r.peak_throughput == 400.0 and r.raw_sample_count == 100
    assert r.p99_latency_ms == 12.0 and r.p50_latency_ms == 10.0
