"""Runs a few plans (for ncu launch lists / --set full captures and
compute-sanitizer runs).

    python tools/profile_one.py [robot] [reps] [single|batch] [n_problems] [workers]

single: one cage problem, prrtc_plan with `workers` CTAs (default 0 = one per SM);
batch:  the first n_problems (default 1000) of the robot's set as one
        device-resident batch at the bench headline's params (workers=1,
        tree_capacity 20000).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else "single"
n_prob = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
workers = int(sys.argv[5]) if len(sys.argv) > 5 else (0 if mode == "single" else 1)
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
params = PlannerParams(workers=workers, tree_capacity=20000)
if mode == "single":
    i = int(np.where(d["kind"] == "cage")[0][0])
    sc = make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0]
    for _ in range(n):
        r = planner.plan(m, sc, d["start"][i], d["goal"][i], params)
        print(r.status.name, r.iterations_total, f"{r.device_time_ms:.3f} ms", r.tree_nodes, r.message)
else:
    idx = np.arange(n_prob) % len(d["pid"])  # (n_prob > 1000 repeats the set)
    scenes0 = [make_scene(robot, str(kk), int(p))[0] for kk, p in zip(d["kind"], d["pid"])]
    ds = [planner.device_scene(sc) for sc in scenes0]
    b = planner.Batch(m, [ds[i] for i in idx], d["start"][idx], d["goal"][idx], params)
    for _ in range(n):
        b.launch()
        res = b.results()
        print("solved", np.mean([r.status == 0 for r in res]), {r.message for r in res if r.message})
