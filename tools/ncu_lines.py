"""Aggregate ncu warp-stall samples per CUDA source line (reads an .ncu-rep)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
agg = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "Function Name") and len(r) > 6:
        try:
            agg.append((float(r[4]), fname, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
for s, f, l, t in sorted(agg, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{l:>5}  {t}")
