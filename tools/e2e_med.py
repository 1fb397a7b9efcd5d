"""Medians of the PRRTC_HOST_TRACE components in a log: python tools/e2e_med.py log"""
import re
import sys
from collections import defaultdict

import numpy as np

vals = defaultdict(list)
for line in open(sys.argv[1]):
    if line.startswith("prrtc host:") or line.startswith("prrtc enqueue:"):
        pre = "enq_" if line.startswith("prrtc enqueue:") else ""
        for k, v in re.findall(r"([a-z_+0-9]+) ([0-9.]+)", line.replace("wait+d2h", "wait_d2h")):
            vals[pre + k].append(float(v))
print(" | ".join(f"{k} {np.median(v):.1f}" for k, v in vals.items()))
