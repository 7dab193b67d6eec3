"""Aggregate an ncu report's per-instruction warp-stall samples by CUDA source line of one
kernel: python tools/ncu_lines.py report.ncu-rep cubin source.cu [top] [first_line last_line].
The cubin must be the one the profiled library was linked from (nvdisasm -g line info)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, src = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lo, hi = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else (0, 10 ** 9)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines, cur = {}, None
for l in dis.splitlines():
    m = re.search(r'//## File ".*", line (\d+)', l)
    if m:
        cur = int(m.group(1))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur is not None:
        lines[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
idx = h.index("Warp Stall Sampling (All Samples)")
agg, base, tot = collections.Counter(), None, 0.0
for r in rows[2:]:
    try:
        a, v = int(r[0], 16), float(r[idx])
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    ln = lines.get(a - base)
    if ln is not None and lo <= ln <= hi:
        agg[ln] += v
        tot += v
text = open(src).read().split("\n")
print(f"samples {tot:.0f} in lines [{lo}, {hi}]")
for ln, v in agg.most_common(top):
    print(f"{v / tot * 100:5.1f}% L{ln}: {text[ln - 1].strip()[:110]}")
