"""Per-phase cycle shares of plan_kernel (PRRTC_TRACE=1): one hard single
problem at several CTA counts, then the 1000-problem batch."""
import os
import sys
from pathlib import Path

import numpy as np

os.environ["PRRTC_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots  # noqa: E402
from paper_2503_06757_b200.model import PlannerParams  # noqa: E402
from paper_2503_06757_b200.scenes import make_scene  # noqa: E402

robot = sys.argv[1] if len(sys.argv) > 1 else "panda"
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / f"problems_{robot}.npz")
m = robots.get(robot)
for i in (400, 700):
    sc = planner.device_scene(make_scene(robot, str(d["kind"][i]), int(d["pid"][i]))[0])
    for w in (1, 32, 296):
        for rep in range(2):
            print(f"--- problem {i} ({d['kind'][i]}) workers {w} rep {rep}", file=sys.stderr, flush=True)
            r = planner.plan(m, sc, d["start"][i], d["goal"][i], PlannerParams(workers=w, tree_capacity=20000))
            print(f"    {r.status.name} dev {r.device_time_ms:.3f} ms iters {r.iterations_total}", file=sys.stderr,
                  flush=True)
scenes = [make_scene(robot, str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
b = planner.Batch(m, scenes, d["start"], d["goal"], PlannerParams(workers=1, tree_capacity=20000))  # bench headline params
for rep in range(2):
    print(f"--- batch rep {rep}", file=sys.stderr, flush=True)
    b.launch()
    res = b.results()
