"""Per-problem timeline of one headline batch (PRRTC_TRACE + PRRTC_DUMP_CTL):
when problems start and finish, and how the CTAs' time splits at the tail.

    python tools/batch_timeline.py [robot] [workers]
"""
import os
import sys
from pathlib import Path

import numpy as np

os.environ["PRRTC_TRACE"] = "1"
os.environ["PRRTC_DUMP_CTL"] = "/tmp/ctl.txt"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
b = planner.Batch(m, scenes, d["start"], d["goal"], PlannerParams(workers=W, tree_capacity=20000))
for rep in range(3):
    b.launch()
    b.results()
t = np.loadtxt("/tmp/ctl.txt")
st, en, it, done = t[:, 1], t[:, 2], t[:, 3], t[:, 4]
print(f"batch end {en.max():.3f} ms; starts: median {np.median(st):.3f} max {st.max():.3f}")
for q in (50, 90, 99, 100):
    print(f"end p{q}: {np.percentile(en, q):.3f} ms")
fail = done == 2
print(f"failed {fail.sum()}: end median {np.median(en[fail]):.3f} max {en[fail].max():.3f}; "
      f"duration median {np.median((en - st)[fail]):.3f}")
print(f"solved: end median {np.median(en[~fail]):.3f}, duration median {np.median((en - st)[~fail]):.3f}, "
      f"iterations median {np.median(it[~fail]):.0f}")
late = np.argsort(en)[-10:]
for i in late:
    print(f"  problem {int(t[i,0])} kind {d['kind'][int(t[i,0])]} start {st[i]:.3f} end {en[i]:.3f} iters {it[i]:.0f} done {int(done[i])}")
