"""Per-CUDA-source-line instructions executed and stall samples of an .ncu-rep."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass,cuda", "--csv"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = None, None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
    elif hdr and r and len(r) == len(hdr) and r[0].isdigit():
        try:
            agg.append((int(r[ie] or 0), int(r[ss] or 0), fname, r[0], r[1].strip()[:90]))
        except ValueError:
            pass
ti = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"total warp instructions {ti}  ({ti / norm:.1f} per unit)")
for a in sorted(agg, key=lambda a: -a[1])[:top]:
    print(f"{a[0] / norm:7.1f}/u {100 * a[1] / ts:5.1f}%smp {a[2]}:{a[3]:>5} {a[4]}")
