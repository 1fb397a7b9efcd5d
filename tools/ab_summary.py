"""Mean batch kernel ms per (robot, setting) from an ab_env.sh / ab_tail.sh log:
    python tools/ab_summary.py gpurun_out/env_VAR/out.txt"""
import collections
import re
import sys

d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"(.*) rep \d+: (\w+):.*kernel ([\d.]+) ms", line)
    if m:
        d[(m.group(2), m.group(1))].append(float(m.group(3)))
for k in sorted(d):
    print(k, d[k], round(sum(d[k]) / len(d[k]), 3))
