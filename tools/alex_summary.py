"""Summarise tools/gpu_alex_prof.sh's launch CSV: per launch of the last step, time, grid,
tensor-pipe activity and DRAM read bytes; totals per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
by = collections.OrderedDict()
for d in data:
    by.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
ids = list(by)
half = ids[len(ids) // 2:]
tot, per = 0.0, collections.defaultdict(float)
verbose = len(sys.argv) > 2
for k in half:
    v = by[k]
    t = float(v["gpu__time_duration.sum"][0].replace(",", ""))
    if v["gpu__time_duration.sum"][1] in ("nsecond", "ns"):
        t /= 1000
    tot += t
    name = v["name"].split("(")[0].replace("dsb::<unnamed>::", "").replace("void ", "")
    per[name] += t
    if verbose:
        g = v.get("launch__grid_size", ("", ""))[0]
        tp = v.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", ("", ""))[0]
        print(f"{t:8.1f} us  grid {g:>6}  tensor {tp:>6}%  {name}")
for n, t in sorted(per.items(), key=lambda x: -x[1]):
    print(f"{t:9.1f} us {100 * t / tot:5.1f}%  {n}")
print(f"total {tot:.1f} us over {len(half)} launches (serialised, cold)")
