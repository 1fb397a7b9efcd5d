"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict

rows = csv.reader(open(sys.argv[1]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
tot = 0
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0].isdigit() and len(r) > 6:
        try:
            samples = int(r[4])
        except ValueError:
            continue
        inst = int(r[7]) if r[7].isdigit() else 0
        agg.append((samples, cur, int(r[0]), r[1].strip()[:90], inst))
        tot += samples
agg.sort(reverse=True)
print(f"total stall samples {tot}")
for s, f, l, src, inst in agg[:n]:
    print(f"{100.0 * s / tot:5.1f}% {f}:{l:<5} inst {inst:>11}  {src}")
