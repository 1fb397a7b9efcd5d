import os, sys
os.environ["PRRTC_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_2503_06757_b200 import planner
from paper_2503_06757_b200.model import PlannerParams
model, scenes, S, G, kinds = bench.load_workload("panda", 1000)
for i in (0, 100, 400, 700, 900):
    sc = planner.device_scene(scenes[i])
    for rep in range(3):
        r = planner.plan(model, sc, S[i], G[i], PlannerParams())
