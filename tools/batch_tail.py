"""Slowest problems of the 1000-problem batch: device span, iterations, status, tree sizes."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402
robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
b = planner.Batch(m, scenes, d["start"], d["goal"], PlannerParams())
for rep in range(2):
    b.launch()
    res = b.results()
dv = np.array([r.device_time_ms for r in res])
order = np.argsort(-dv)[:15]
for i in order:
    r = res[i]
    print(f"problem {i} {d['kind'][i]}: {r.status.name} dev {r.device_time_ms:.3f} ms iters {r.iterations_total} "
          f"nodes {r.tree_nodes} {r.message}")
print("time-sorted spans:", np.round(np.sort(dv)[-30:], 2))
