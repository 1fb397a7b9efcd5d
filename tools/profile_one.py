"""Runs a few single-problem plans (for ncu launch lists / --set full captures)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams
from paper_2503_06757_b200.scenes import make_scene

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else "single"
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
params = PlannerParams(tree_capacity=20000)
if mode == "single":
    i = int(np.where(d["kind"] == "cage")[0][0])
    sc = make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0]
    for _ in range(n):
        r = planner.plan(m, sc, d["start"][i], d["goal"][i], params)
        print(r.status.name, r.iterations_total, f"{r.device_time_ms:.3f} ms", r.tree_nodes)
else:
    scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
    b = planner.Batch(m, scenes, d["start"], d["goal"], params)
    for _ in range(n):
        b.launch()
        res = b.results()
        print("solved", np.mean([r.status == 0 for r in res]))
