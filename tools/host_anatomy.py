"""Host-side anatomy of single-problem prrtc_plan calls (PRRTC_HOST_TRACE):
median of each component over n calls.  python tools/host_anatomy.py [n]"""
import os
import re
import subprocess
import sys
from pathlib import Path

if os.environ.get("_HA_CHILD") != "1":
    env = dict(os.environ, _HA_CHILD="1", PRRTC_HOST_TRACE="1")
    p = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    import numpy as np
    enq = [list(map(float, m)) for m in re.findall(
        r"prrtc enqueue: copies ([\d.]+) ev0 ([\d.]+) launch ([\d.]+) ev1 ([\d.]+) us", p.stderr)]
    host = [list(map(float, m)) for m in re.findall(
        r"prrtc host: setup ([\d.]+) bind ([\d.]+) enqueue ([\d.]+) wait\+d2h ([\d.]+) fill ([\d.]+) us \| "
        r"kernel ([\d.]+) problem ([\d.]+) us", p.stderr)]
    print(p.stdout.strip())
    if enq:
        e = np.median(np.array(enq[10:]), axis=0)
        print("enqueue (us): copies %.1f ev0 %.1f launch %.1f ev1 %.1f" % tuple(e))
    if host:
        h = np.median(np.array(host[10:]), axis=0)
        print("call (us): setup %.1f bind %.1f enqueue %.1f wait %.1f fill %.1f | kernel events %.1f problem %.1f" % tuple(h))
    sys.exit(0)

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "problems_panda.npz")
m = robots.get("panda")
rob = planner.device_robot(m)
idx = np.linspace(0, 999, n).astype(int)
scs = [planner.device_scene(make_scene("panda", str(d["kind"][i]), int(d["pid"][i]))[0]) for i in idx]
walls = []
for k, i in enumerate(idx):
    r = planner.plan(rob, scs[k], d["start"][i], d["goal"][i], PlannerParams())
    walls.append(r.wall_time_ms)
print(f"wall median {np.median(walls[10:]) * 1e3:.1f} us over {len(walls) - 10} calls")
