import os, sys
os.environ["PRRTC_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np
from pathlib import Path
from paper_2503_06757_b200 import planner, robots
from paper_2503_06757_b200.model import PlannerParams
from paper_2503_06757_b200.scenes import make_scene
d = np.load("/root/repo/tests/golden/problems_baxter.npz")
m = robots.get("baxter")
scenes = [make_scene("baxter", str(k), int(p))[0] for k, p in zip(d["kind"], d["pid"])]
b = planner.Batch(m, scenes, d["start"], d["goal"], PlannerParams(dd_radius=4.0))
for rep in range(2):
    print(f"--- batch rep {rep}", file=sys.stderr, flush=True)
    b.launch(); b.results()
