"""Summarise an ncu launch list (gpu__time_duration + dram bytes) for one forward."""
import collections, csv, json, sys
path, out_summary, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]
ki, mi, vi, ii, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID', 'Metric Unit'))
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3,
         'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = launch.setdefault(int(r[ii]), {'name': r[ki]})
    d[r[mi]] = float(r[vi].replace(',', '')) * scale.get(r[ui], 1)
L = list(launch.values())
starts = [i for i, d in enumerate(L) if 'input_pack' in d['name']]
fwd = L[starts[-3]:starts[-2]]
fwd = [d for d in fwd if 'gen_normal' not in d['name']]
tot = sum(d['gpu__time_duration.sum'] for d in fwd)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in fwd:
    a = agg[d['name'].split('(')[0].replace('void ', '')]
    a[0] += 1
    a[1] += d['gpu__time_duration.sum']
    a[2] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
lines = [f"{k:50s} launches={n:3d} time={us:9.1f} us share={100 * us / tot:5.1f}%  dram={by / 1e6:9.1f} MB"
         for k, (n, us, by) in sorted(agg.items(), key=lambda x: -x[1][1])]
FAMILY = ('tc_gemm', 'conv_band', 'chain_gemm', 'stem_pool')   # the tcgen05 conv/GEMM kernels
tc = [d for d in fwd if any(f in d['name'] for f in FAMILY)]
tb = sum(d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0) for d in tc) / len(tc)
share = sum(d['gpu__time_duration.sum'] for d in tc) / tot
head = (f"one ResNet-50 bf16 batch-256 forward from the ncu launch list (cold cache, serialised: "
        f"compare shares, not absolutes)\ntotal {tot:.1f} us over {len(fwd)} launches; "
        f"tcgen05 conv/GEMM share {100 * share:.1f}%, avg DRAM traffic per launch {tb / 1e6:.1f} MB\n")
open(out_summary, 'w').write(head + "\n".join(lines) + "\n")
json.dump({"model": "resnet50", "batch": 256, "tcgen05_bytes_per_launch": tb, "tcgen05_launches_per_forward": len(tc),
           "tcgen05_time_share_ncu": share, "family": list(FAMILY), "forward_us_ncu": tot,
           "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     "--clock-control none, python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu"},
          open(out_json, 'w'), indent=1)
print(head + "\n".join(lines))
