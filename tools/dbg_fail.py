import os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams
from paper_2503_06757_b200.scenes import make_scene
d = np.load("tests/golden/problems_panda.npz")
m = robots.get("panda")
i = 700
sc = planner.device_scene(make_scene("panda", str(d["kind"][i]), int(d["pid"][i]))[0])
for w in (32, 64, 148, 296):
    for rep in range(3):
        r = planner.plan(m, sc, d["start"][i], d["goal"][i], PlannerParams(workers=w, tree_capacity=20000))
        print(os.environ.get("PRRTC_DEBUG_FLAGS"), w, r.status.name, f"{r.device_time_ms:.3f}", r.iterations_total, r.tree_nodes, r.message, flush=True)
