"""Top CUDA source lines of an ncu report by warp-stall samples (captured
with --import-source on, code built with -lineinfo).

    python tools/ncu_top_lines.py <report.ncu-rep> [n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, ci = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ci = {}
        for i, k in enumerate(r):
            ci.setdefault(k, i)
        continue
    if ci is None or r[0] in ("", "Function Name") or not r[0].isdigit():
        continue
    try:
        samp = float(r[4] or 0)
        inst = float(r[7] or 0)
    except ValueError:
        continue
    rows.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(x[0] for x in rows) or 1
print(f"total stall samples {tot:.0f}")
for s, i, loc, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% {loc:26s} inst {i:11.0f}  {src}")
