"""Per-launch table of one ResNet-50 bf16 b=256 forward from an ncu metrics
CSV (tools/r2_ncu*.sh): duration, tensor-pipe activity, DRAM bytes and GB/s,
L2->SM (xbar) bytes, and the algorithmic roofline fraction of each launch
(HBM: DRAM bytes / duration vs the measured copy bandwidth; the tensor
fraction is ncu's tensor-pipe activity).

    python tools/ncu_launch_table.py gpurun_out/r2_launch_metrics2.csv profiles/r2_launch_table.txt
"""
import collections
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                "ID", "Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    return list(launches.values())


def main():
    src, out = sys.argv[1], sys.argv[2]
    L = load(src)
    # one forward = from the last input-packing launch (images) or token pack (BERT)
    first = sys.argv[3] if len(sys.argv) > 3 else None
    starts = [i for i, d in enumerate(L)
              if (first and first in d["name"]) or (not first and ("input_pack" in d["name"]
                                                                     or "tokens_pack" in d["name"]))]
    fwd = L[starts[-1]:]
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    tf_peak, hbm_peak = pk["bf16_tflops"], pk["hbm_gbs"]
    lines = [f"ncu --metrics (cold cache, serialised) of one forward: "
             f"{src}\npeaks: bf16 {tf_peak} TFLOP/s burst, HBM {hbm_peak} GB/s "
             f"(MEASURED_PEAKS.json)\n",
             f"{'#':>2} {'kernel':34s} {'us':>7s} {'tensor%':>7s} {'DRAM MB':>8s} {'GB/s':>6s} "
             f"{'HBM frac':>8s} {'xbar MB':>8s}"]
    tot = 0.0
    by = collections.defaultdict(float)
    for i, d in enumerate(fwd):
        us = d["gpu__time_duration.sum"]
        tot += us
        dram = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        gbs = dram / us / 1e3
        name = d["name"].split("(")[0].replace("void ", "").replace("b2::", "")[:34]
        by[name.split("<")[0]] += us
        lines.append(f"{i:2d} {name:34s} {us:7.1f} "
                     f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):7.1f} "
                     f"{dram / 1e6:8.1f} {gbs:6.0f} {gbs / hbm_peak:8.2f} "
                     f"{d.get('l1tex__m_xbar2l1tex_read_bytes.sum', 0) / 1e6:8.1f}")
    lines.append(f"\ntotal {tot:.1f} us over {len(fwd)} launches")
    for k, us in sorted(by.items(), key=lambda x: -x[1]):
        lines.append(f"  {k:30s} {us:8.1f} us  {100 * us / tot:5.1f}%")
    Path(out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
