"""Warp-stall samples per CUDA source line of one kernel in an .ncu-rep (needs -lineinfo)."""
import collections
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, agg, src = None, collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        v = int(r[4] or 0)
    except (ValueError, IndexError):
        continue
    agg[(fname, int(r[0]))] += v
    src[(fname, int(r[0]))] = r[1][:90]
tot = sum(agg.values()) or 1
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]}  {src[k]}")
