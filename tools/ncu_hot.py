"""Hot SASS lines of an ncu source page (csv): the lines holding most warp-stall
samples, with their neighbours' role tags.  usage: ncu_hot.py <src.csv> [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ia, isrc, iall, inot, iex = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                  "Warp Stall Sampling (Not-issued Samples)",
                                                  "Instructions Executed"))
body = [r for r in rows[2:] if len(r) > iex]
tot = sum(float(r[iall] or 0) for r in body)
print(f"{len(body)} SASS lines, {tot:.0f} stall samples")
for k, r in sorted(enumerate(body), key=lambda kr: -float(kr[1][iall] or 0))[:n]:
    print(f"{k:5d} {float(r[iall] or 0) / tot * 100:5.1f}% notiss {float(r[inot] or 0) / tot * 100:5.1f}% "
          f"exec {r[iex]:>9s}  {r[isrc][:90]}")
