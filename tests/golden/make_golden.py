"""Generate golden vectors from the REFERENCE implementation (run in the dev
container where /root/reference exists; the outputs are committed so the GPU
box, which has no /root/reference, can check against them).

    python tests/golden/make_golden.py

* stats_golden.json  — reference profiler/stats.py percentile / peak_throughput
  / aggregate on seeded random inputs plus the reference tests' known answers
  (pkg/tests/test_stats.py:20-114).
* toy_codec.json     — reference converter/toyformat.py encodings (hex) and
  canonical JSON of seeded random graphs (pkg/tests/test_toyformat.py:13-36).
* mlp_golden.json    — the C1 MLP (seed 0) toy-binary digest + fp64 logits of
  oracle/toyref.c on 4 seeded inputs (cross-checks the numpy oracle).
"""
import hashlib
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parent.parent))

from modelci.profiler.stats import LatencySamples, ResourceSample, aggregate, peak_throughput, percentile  # noqa: E402
from modelci.converter import toyformat as ref_toy  # noqa: E402


def stats_golden():
    rng = random.Random(0x5EED)
    pct, thr, agg = [], [], []
    for _ in range(400):
        n = rng.randint(1, 60)
        s = [rng.randint(-1000, 1000) for _ in range(n)]
        p = rng.choice([rng.randint(1, 100), 97.5, 99.9, 50.0, 0.1])
        pct.append({"samples": s, "p": p, "out": percentile(s, p)})
    for _ in range(300):
        n = rng.randint(1, 80)
        ts = [round(rng.uniform(0.5, 4000), 3) for _ in range(n)]
        b = rng.randint(1, 16)
        w = rng.choice([250, 500, 1000, 2000])
        thr.append({"ts": ts, "batch": b, "window": w, "out": peak_throughput(ts, b, w)})
    for _ in range(40):
        n = rng.randint(1, 200)
        lat = [round(rng.uniform(0.01, 50), 4) for _ in range(n)]
        comp = sorted(round(rng.uniform(0.1, 3000), 3) for _ in range(n))
        trace = [[i * 100.0, rng.random(), rng.randint(1, 10**9)] for i in range(rng.randint(0, 12))]
        b = rng.randint(1, 256)
        r = aggregate(LatencySamples(lat, comp), [ResourceSample(*t) for t in trace], b,
                      variant_id="v", device="gpu:0", backend="b200", protocol="grpc-style",
                      resource_scope="gpu:0")
        d = r.to_doc()
        d.pop("measured_at")
        agg.append({"lat": lat, "comp": comp, "trace": trace, "batch": b, "out": d})
    known = {"steady": peak_throughput([10 * i for i in range(1, 201)], 4),
             "short": peak_throughput([500], 1),
             "bursty": peak_throughput([5 + 10 * i for i in range(100)] +
                                       [1010 + 20 * i for i in range(50)], 1),
             "p95_1_100": percentile(list(range(1, 101)), 95),
             "p50_three": percentile([10, 20, 30], 50)}
    return {"percentile": pct, "peak_throughput": thr, "aggregate": agg, "known": known}


def random_graph(rng):
    layers = []
    for _ in range(rng.randint(1, 6)):
        i, o = rng.randint(1, 8), rng.randint(1, 8)
        w = [rng.uniform(-10, 10) for _ in range(i * o)] if rng.random() < 0.8 else []
        layers.append({"op": rng.choice(["linear", "relu", "norm", "gelu"]), "in_dim": i,
                       "out_dim": o, "weights": w})
    return {"layers": layers}


def toy_golden():
    rng = random.Random(0xF00D)
    out = []
    for _ in range(60):
        g = random_graph(rng)
        out.append({"graph": g, "binary_hex": ref_toy.encode_binary(g).hex(),
                    "canonical": ref_toy.canonical_json(g).decode()})
    return out


def mlp_golden():
    import numpy as np
    from paper_2006_05096_b200 import zoo
    sys.path.insert(0, str(HERE.parent.parent / "oracle"))
    import toyref
    g = zoo.make_mlp_graph(0)
    blob = ref_toy.encode_binary(g)
    x = np.random.default_rng(7).standard_normal((4, 784))
    y = toyref.forward(blob, x)
    return {"seed": 0, "toy_binary_sha256": hashlib.sha256(blob).hexdigest(),
            "x_seed": 7, "logits": y.tolist()}


if __name__ == "__main__":
    (HERE / "stats_golden.json").write_text(json.dumps(stats_golden()))
    (HERE / "toy_codec.json").write_text(json.dumps(toy_golden()))
    (HERE / "mlp_golden.json").write_text(json.dumps(mlp_golden()))
    print("golden vectors written")
