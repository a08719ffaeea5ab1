"""Key counters of ncu --set full captures -> a text summary (profiles/)."""
import csv, subprocess, sys
KEYS = [("gpu__time_duration.sum", "duration us"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
        ("dram__bytes_read.sum", "DRAM read MB"), ("dram__bytes_write.sum", "DRAM write MB"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("launch__registers_per_thread", "registers/thread"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block")]
out = [sys.argv[1]]
for rep in sys.argv[3:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, v = rows[0], rows[2]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else rep
    out.append(f"\n== {name[:110]}")
    for k, label in KEYS:
        if k in h:
            out.append(f"   {label:24s} {v[h.index(k)]}")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out))
