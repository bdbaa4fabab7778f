"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per
kernel launch count, total / mean time and share (cold-cache, serialised:
compare shares, not absolutes)."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
only = sys.argv[2] if len(sys.argv) > 2 else "cw::"
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg = defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum" or only not in r[ki]:
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] in ("usecond", "us") else (v / 1e6 if r[ui] in ("nsecond", "ns") else v)   # -> ms
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values()) or 1.0
print(f"{'kernel':44s} {'n':>5s} {'sum ms':>10s} {'avg us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:44s} {len(v):5d} {sum(v):10.3f} {1e3 * sum(v) / len(v):10.1f} {sum(v) / tot:6.3f}")
