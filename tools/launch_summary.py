"""Summarise an ncu --metrics gpu__time_duration.sum CSV: time per kernel name over the
last `frac` of the launches (default: the second half = the last of two steps)."""
import collections
import csv
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
data = data[int(len(data) * (1 - frac)):]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    t = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    name = d["Kernel Name"].split("(")[0][-60:]
    agg[name][0] += 1
    agg[name][1] += t
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}% {v[0]:4d}x  {k}")
print(f"total {tot:.1f} us over {len(data)} launches")
