"""Single-problem timing breakdown (PRRTC_TRACE) for several CTA counts."""
import os, sys
from pathlib import Path
import numpy as np
os.environ["PRRTC_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams
from paper_2503_06757_b200.scenes import make_scene
d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "problems_panda.npz")
m = robots.get("panda")
i = 400
sc = planner.device_scene(make_scene("panda", str(d["kind"][i]), int(d["pid"][i]))[0])
for w in (32, 148, 296, 592):
    for rep in range(3):
        r = planner.plan(m, sc, d["start"][i], d["goal"][i], PlannerParams(workers=w, tree_capacity=20000))
        print(f"workers {w}: wall {r.wall_time_ms:.3f} dev {r.device_time_ms:.3f} iters {r.iterations_total}", file=sys.stderr, flush=True)
