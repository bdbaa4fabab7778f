"""Per-SASS-instruction stall summary of an .ncu-rep (one kernel): totals by
stall reason and the top instructions with their dominant reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kern = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"]
if kern:
    cmd += ["-k", kern]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        recs.append(r)
cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
tot = {hdr[i]: 0 for i in cols}
allsamp = 0
for r in recs:
    allsamp += int(r[2] or 0)
    for i in cols:
        tot[hdr[i]] += int(r[i] or 0)
print("total samples", allsamp)
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:28s} {v:8d} {100*v/max(allsamp,1):5.1f}%")
print()
idx = {r[0]: n for n, r in enumerate(recs)}
for n, r in sorted(enumerate(recs), key=lambda t: -int(t[1][2] or 0))[:top]:
    s = int(r[2] or 0)
    why = sorted(((int(r[i] or 0), hdr[i][6:]) for i in cols), reverse=True)[:2]
    print(f"{100*s/max(allsamp,1):5.1f}% #{n:5d} {r[1].strip()[:60]:60s} {why}")
